cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in variants/nodelta.so libewbem_b200.so; do
  timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v
done
done > gpurun_out/mf2_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/mf2_tests.log 2>&1; echo tests_rc=$?
