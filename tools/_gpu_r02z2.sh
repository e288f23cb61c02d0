set -x
mkdir -p gpurun_out
timeout 600 python tools/pi_time.py 5 auto,ws3,ws7 > gpurun_out/r02z2_pi_time.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_pi.py -q -x > gpurun_out/r02z2_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02z2_pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pi_ws_kernel -s 1 -c 1 -o gpurun_out/r02z2_piws python tools/prof_launch.py pi 30000 720 > gpurun_out/r02z2_ncu_piws.log 2>&1
