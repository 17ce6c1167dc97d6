cd $GRAFT_REPO_ROOT
export ASM_QUICK=1
for rep in 1 2; do
for v in variants/old.so variants/new.so variants/exact.so libewbem_b200.so; do
  timeout 300 python tools/asm_multi_time.py paper_1212_3032_b200/$v
done
done > gpurun_out/far3_ab.log 2>&1
for v in variants/semglob.so libewbem_b200.so; do timeout 300 python tools/sem_time.py paper_1212_3032_b200/$v; done > gpurun_out/far3_sem.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_solvers.py -m gpu -q -x --deselect tests/test_gpu_solvers.py::test_cfg2_stepwise_all_frequencies > gpurun_out/far3_tests.log 2>&1; echo tests_rc=$?
timeout 300 python tools/sweep_time.py > gpurun_out/far3_sweep.log 2>&1
