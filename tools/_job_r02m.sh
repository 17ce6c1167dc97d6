cd $GRAFT_REPO_ROOT
python tools/prof_mf.py 5 > gpurun_out/r02m_plain_mf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mf_farmid -c 1 -o gpurun_out/r02m_mf python tools/prof_mf.py 5 > gpurun_out/r02m_ncu_mf.log 2>&1; echo mf_rc=$?
python tools/prof_multi.py > gpurun_out/r02m_plain_multi.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_far_multi -c 1 -o gpurun_out/r02m_far python tools/prof_multi.py > gpurun_out/r02m_ncu_far.log 2>&1; echo far_rc=$?
