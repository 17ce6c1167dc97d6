cd $GRAFT_REPO_ROOT
EWB_LIBRARY=$PWD/paper_1212_3032_b200/variants/debug.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02v_gpu_debug.log 2>&1; echo dbg_rc=$?
B="python bench.py --steps 1 --warmup 1"
$B > gpurun_out/r02v_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02v_launches.csv $B > gpurun_out/r02v_ncu_bench.log 2>&1; echo launches_rc=$?
python tools/prof_cfg2.py 6 > gpurun_out/r02v_plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gmres_f -s 5 -c 1 -o gpurun_out/r02v_gmres python tools/prof_cfg2.py 6 > gpurun_out/r02v_ncu_gmres.log 2>&1; echo gmres_rc=$?
python tools/prof_multi.py > gpurun_out/r02v_plain_multi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_far_multi -c 1 -o gpurun_out/r02v_far python tools/prof_multi.py > gpurun_out/r02v_ncu_far.log 2>&1; echo far_rc=$?
