cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/head_gpu.log 2>&1; echo gpu_rc=$?
timeout 120 python __graft_entry__.py smoke > gpurun_out/head_smoke.log 2>&1; echo smoke_rc=$?
start=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/head_bench.log 2>&1; echo bench_rc=$? bench_s=$(( $(date +%s) - start ))
B="python bench.py --steps 1 --warmup 1"
$B > gpurun_out/head_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/head_launches.csv $B > gpurun_out/head_ncu_bench.log 2>&1; echo launches_rc=$?
python tools/prof_multi.py > gpurun_out/head_plain_multi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_far_multi -c 1 -o gpurun_out/head_far python tools/prof_multi.py > gpurun_out/head_ncu_far.log 2>&1; echo far_rc=$?
python tools/sem_time.py > gpurun_out/head_sem_time.log 2>&1; echo sem_rc=$?
