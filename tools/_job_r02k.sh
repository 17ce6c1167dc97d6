cd $GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 1"
$B > gpurun_out/r02k_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02k_launches.csv $B > gpurun_out/r02k_ncu_bench.log 2>&1; echo launches_rc=$?
python tools/prof_cfg2.py 6 > gpurun_out/r02k_plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gmres_f -s 2 -c 1 -o gpurun_out/r02k_gmres python tools/prof_cfg2.py 6 > gpurun_out/r02k_ncu_gmres.log 2>&1; echo gmres_rc=$?
python tools/prof_multi.py > gpurun_out/r02k_plain_multi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_far_multi -c 1 -o gpurun_out/r02k_far python tools/prof_multi.py > gpurun_out/r02k_ncu_far.log 2>&1; echo far_rc=$?
python tools/prof_mf.py 5 > gpurun_out/r02k_plain_mf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mf_farmid -c 1 -o gpurun_out/r02k_mf python tools/prof_mf.py 5 > gpurun_out/r02k_ncu_mf.log 2>&1; echo mf_rc=$?
