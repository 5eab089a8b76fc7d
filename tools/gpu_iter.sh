# one development iteration on the GPU: tests, bench cfg3, ncu of the sweep kernel (every step time-limited;
# profiling only if the tests passed: ncu on a faulting program can wedge the GPU)
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest=$rc
tail -3 gpurun_out/pytest_gpu.log
[ $rc -ne 0 ] && exit 1
timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.log 2>&1; echo b3=$?
grep -o '"time_to_tol_ms": [0-9.]*\|"sweep_ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"sweeps": [0-9.]*' gpurun_out/bench_cfg3.log
bash tools/gpu_prof.sh 3
