cd $GRAFT_REPO_ROOT
for rep in 1 2; do
EWB_LIBRARY=paper_1212_3032_b200/variants/pk1.so timeout 300 python bench.py --workload cfg3 --steps 3 --warmup 1
timeout 300 python bench.py --workload cfg3 --steps 3 --warmup 1
done > gpurun_out/pk_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py tests/test_gpu_assembly.py -m gpu -q -x > gpurun_out/pk_tests.log 2>&1; echo tests_rc=$?
for rep in 1 2; do
for v in variants/nodelta.so libewbem_b200.so; do
  timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v
done
done > gpurun_out/pk_mf.log 2>&1
