# GPU check: tests, smoke, short benches (run under gpurun from the repo root)
set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/smoke.log
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo b2=$?
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo b3=$?
tail -c 1500 gpurun_out/bench_cfg3.log
