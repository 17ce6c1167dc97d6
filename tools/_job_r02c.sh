set -x
cd $GRAFT_REPO_ROOT
timeout 900 python tools/cfg1_drift.py > gpurun_out/r02c_drift.json 2> gpurun_out/r02c_drift.err
echo drift_rc=$?
for tool in memcheck racecheck synccheck; do
  for m in dense matfree gemv; do
    timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py $m > gpurun_out/r02c_san_${tool}_${m}.log 2>&1
    echo san_${tool}_${m}_rc=$?
  done
done
