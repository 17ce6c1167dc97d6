cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/final_gpu.log 2>&1; echo gpu_rc=$?
timeout 120 python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$?
start=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.log 2>&1; echo bench_rc=$? bench_s=$(( $(date +%s) - start ))
start=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_ref.log 2>&1; echo ref_rc=$? ref_s=$(( $(date +%s) - start ))
