set -x
mkdir -p gpurun_out/s7
python scripts/profile_filter_call.py 20000 26 3 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma -s 3 -c 1 -o gpurun_out/s7/filter_k26_bsum python scripts/profile_filter_call.py 20000 26 3 > gpurun_out/s7/ncu26.log 2>&1; echo ncu_rc=$?
python scripts/profile_filter_call.py 20000 51 3 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_tma -s 3 -c 1 -o gpurun_out/s7/filter_k51_bsum python scripts/profile_filter_call.py 20000 51 3 > gpurun_out/s7/ncu51.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/s7
