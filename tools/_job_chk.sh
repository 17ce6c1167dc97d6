cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_solvers.py -m gpu -q -x -k "ring_staged or sem" > gpurun_out/chk_tests.log 2>&1; echo tests_rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/chk_bench.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --workload cfg1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/chk_bench_cfg1.log 2>&1; echo cfg1_rc=$?
