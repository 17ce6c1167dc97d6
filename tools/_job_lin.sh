cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in libewbem_b200.so variants/lin.so; do timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v; done
done > gpurun_out/lin_mf.log 2>&1
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/lin.so timeout 900 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q -x -k "cfg5 or matfree or operator" > gpurun_out/lin_tests.log 2>&1; echo tests_rc=$?
