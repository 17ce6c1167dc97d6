cd $GRAFT_REPO_ROOT
for v in paper_1212_3032_b200/variants/head.so paper_1212_3032_b200/libewbem_b200.so paper_1212_3032_b200/variants/far128x4.so paper_1212_3032_b200/variants/far64x7.so paper_1212_3032_b200/variants/far64x6.so; do
  timeout 300 python tools/asm_multi_time.py $v
done > gpurun_out/far_variants.log 2>&1
timeout 600 python -m pytest tests/test_gpu_assembly.py -m gpu -q > gpurun_out/far_asm_tests.log 2>&1; echo asm_rc=$?
