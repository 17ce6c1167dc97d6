cd $GRAFT_REPO_ROOT
export ASM_QUICK=1
for rep in 1 2; do
for v in old new newcb new4 newcb4; do
  timeout 300 python tools/asm_multi_time.py paper_1212_3032_b200/variants/$v.so
done
done > gpurun_out/far2_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_assembly.py -m gpu -q -x > gpurun_out/far2_tests.log 2>&1; echo tests_rc=$?
for nb in 8 16 32; do EWB_ASSEMBLY_BATCH=$nb timeout 300 python tools/sweep_time.py; done > gpurun_out/far2_batch.log 2>&1
