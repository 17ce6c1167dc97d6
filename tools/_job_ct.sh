cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in variants/ctas64.so variants/ctas128.so variants/ctas256.so; do timeout 300 python tools/mf_time.py 6 paper_1212_3032_b200/$v; done
done > gpurun_out/ct2_mf.log 2>&1
for v in variants/ctas64.so variants/ctas256.so; do timeout 300 python tools/mf_time.py 4 paper_1212_3032_b200/$v; done > gpurun_out/ct2_mf4.log 2>&1
