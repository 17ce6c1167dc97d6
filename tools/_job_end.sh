cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/end_gpu.log 2>&1; echo gpu_rc=$?
timeout 120 python __graft_entry__.py smoke > gpurun_out/end_smoke.log 2>&1; echo smoke_rc=$?
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/debug.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/end_gpu_debug.log 2>&1; echo dbg_rc=$?
start=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/end_bench.log 2>&1; echo bench_rc=$? bench_s=$(( $(date +%s) - start ))
start=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/end_ref.log 2>&1; echo ref_rc=$? ref_s=$(( $(date +%s) - start ))
B="python bench.py --steps 1 --warmup 1"
$B > gpurun_out/end_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/end_launches.csv $B > gpurun_out/end_ncu_bench.log 2>&1; echo launches_rc=$?
python tools/prof_cfg2.py 6 > gpurun_out/end_plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gmres_f -s 5 -c 1 -o gpurun_out/end_gmres python tools/prof_cfg2.py 6 > gpurun_out/end_ncu_gmres.log 2>&1; echo gmres_rc=$?
python tools/prof_multi.py > gpurun_out/end_plain_multi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_far_multi -c 1 -o gpurun_out/end_far python tools/prof_multi.py > gpurun_out/end_ncu_far.log 2>&1; echo far_rc=$?
python tools/prof_mf.py > gpurun_out/end_plain_mf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mf_farmid -c 1 -o gpurun_out/end_mf python tools/prof_mf.py > gpurun_out/end_ncu_mf.log 2>&1; echo mf_rc=$?
python tools/sem_time.py > gpurun_out/end_sem_time.log 2>&1; echo sem_rc=$?
timeout 600 python tools/cfg5_probe.py 33 > gpurun_out/end_cfg5_sweep.log 2>&1; echo cfg5_rc=$?
for w in cfg1 cfg3 cfg4; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/end_bench_$w.log 2>&1; done
