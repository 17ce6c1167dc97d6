cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 300 python bench.py --workload cfg3 --steps 3 --warmup 1
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/pk16.so timeout 300 python bench.py --workload cfg3 --steps 3 --warmup 1
done > gpurun_out/pk2_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_matfree.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/pk2_tests.log 2>&1; echo tests_rc=$?
timeout 600 python tools/cfg5_probe.py 33 > gpurun_out/pk2_cfg5_sweep.log 2>&1; echo cfg5_rc=$?
