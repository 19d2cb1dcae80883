set -x
mkdir -p gpurun_out/s10
(time timeout 2400 python -m pytest tests -m gpu -x -q) > gpurun_out/s10/pytest.log 2>&1; echo rc=$?
tail -5 gpurun_out/s10/pytest.log
timeout 900 python scripts/rank_phase_probe.py > gpurun_out/s10/rank_phases.json 2> gpurun_out/s10/rank_phases.err; echo rc=$?
