cd $GRAFT_REPO_ROOT
for v in paper_1212_3032_b200/variants/head.so paper_1212_3032_b200/libewbem_b200.so; do
  timeout 300 python tools/asm_multi_time.py $v
done > gpurun_out/ab_far.log 2>&1
for v in paper_1212_3032_b200/variants/head.so paper_1212_3032_b200/libewbem_b200.so; do
  timeout 300 python tools/mf_time.py 6 $v
done > gpurun_out/ab_mf.log 2>&1
timeout 900 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_matfree.py -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?
