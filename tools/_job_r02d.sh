cd $GRAFT_REPO_ROOT
free -g > gpurun_out/r02d_free.txt; nproc >> gpurun_out/r02d_free.txt; df -h /dev/shm /tmp >> gpurun_out/r02d_free.txt
timeout 600 python tools/diag_cfg1_k.py 4 5 41 > gpurun_out/r02d_diag.json 2> gpurun_out/r02d_diag.err; echo diag_rc=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02d_bench.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02d_ref.log 2>&1; echo ref_rc=$?
