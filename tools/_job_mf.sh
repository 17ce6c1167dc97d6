cd $GRAFT_REPO_ROOT
for v in paper_1212_3032_b200/variants/head.so paper_1212_3032_b200/libewbem_b200.so; do
  timeout 300 python tools/mf_time.py 6 $v
  timeout 300 python tools/mf_time.py 6 $v
done > gpurun_out/mf_variants.log 2>&1
timeout 300 python tools/asm_multi_time.py paper_1212_3032_b200/libewbem_b200.so >> gpurun_out/mf_variants.log 2>&1
timeout 900 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q > gpurun_out/mf_tests.log 2>&1; echo mf_rc=$?
