set -x
mkdir -p gpurun_out/s6
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/s6/pytest_kernels.log 2>&1; echo rc=$?
timeout 900 python scripts/rank_phase_probe.py > gpurun_out/s6/rank_phases.json 2> gpurun_out/s6/rank_phases.err; echo rc=$?
timeout 900 python bench.py --legs tail --steps 3 --warmup 3 > gpurun_out/s6/bench_tail.log 2>&1; echo rc=$?
tail -3 gpurun_out/s6/pytest_kernels.log
