cd $GRAFT_REPO_ROOT
export ASM_QUICK=1
for rep in 1 2; do
for v in variants/rows2.so variants/rows8.so libewbem_b200.so; do
  timeout 300 python tools/asm_multi_time.py paper_1212_3032_b200/$v
done
done > gpurun_out/x_rows.log 2>&1
for nb in 16 32; do EWB_ASSEMBLY_BATCH=$nb timeout 600 python bench.py --steps 4 --warmup 3 --no-cfg5 --no-cpu-baseline; done > gpurun_out/x_batch.log 2>&1
timeout 300 python tools/setup_time.py > gpurun_out/x_setup.log 2>&1
