set -x
mkdir -p gpurun_out/s11
(time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5) > gpurun_out/s11/bench_ref.log 2>&1; echo ref_rc=$?
(time python bench.py --gpus 1 --steps 20 --warmup 5) > gpurun_out/s11/bench.log 2>&1; echo bench_rc=$?
