cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in variants/accbr.so libewbem_b200.so; do timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v; done
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/accbr.so timeout 300 python tools/mf_mask_time.py 6
timeout 300 python tools/mf_mask_time.py 6
done > gpurun_out/acc_mf.log 2>&1
timeout 900 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q -x -k "cfg5 or matfree or operator" > gpurun_out/acc_tests.log 2>&1; echo tests_rc=$?
