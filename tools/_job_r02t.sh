cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02t_gpu.log 2>&1; echo gpu_rc=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02t_bench.log 2>&1; echo bench_rc=$?
timeout 120 python __graft_entry__.py smoke > gpurun_out/r02t_smoke.log 2>&1; echo smoke_rc=$?
