cd $GRAFT_REPO_ROOT
export ASM_QUICK=1
for rep in 1 2; do
for v in new f_base f_mc f_orf f_rp f_mcorf; do
  timeout 300 python tools/asm_multi_time.py paper_1212_3032_b200/variants/$v.so
done
done > gpurun_out/far4_ab.log 2>&1
