cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/chk_gpu.log 2>&1; echo gpu_rc=$?
timeout 120 python __graft_entry__.py smoke > gpurun_out/chk_smoke.log 2>&1; echo smoke_rc=$?
start=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/chk_bench.log 2>&1; echo bench_rc=$? bench_s=$(( $(date +%s) - start ))
