cd $GRAFT_REPO_ROOT
for rep in 1 2; do
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/ysoff.so timeout 300 python tools/mf_mask_time.py 6
timeout 300 python tools/mf_mask_time.py 6
done > gpurun_out/ys_mask.log 2>&1
for v in variants/ysoff.so libewbem_b200.so; do timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v; done > gpurun_out/ys_mf.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/ys_tests.log 2>&1; echo tests_rc=$?
timeout 300 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -k "deep_history or operator" > gpurun_out/ys_tests2.log 2>&1; echo tests2_rc=$?
