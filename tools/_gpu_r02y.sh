set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pi.py -q -x > gpurun_out/r02y_pytest_pi.txt 2>&1; echo "rc=$?" >> gpurun_out/r02y_pytest_pi.txt
timeout 600 python tools/pi_time.py 5 auto,lanes,ws3,ws7 > gpurun_out/r02y_pi_time.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pi_ws_kernel -s 1 -c 1 -o gpurun_out/r02y_piws python tools/prof_launch.py pi 30000 720 > gpurun_out/r02y_ncu_piws.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pi_kernel -s 1 -c 1 -o gpurun_out/r02y_pilanes env NMPCMC_PI_KERNEL=lanes python tools/prof_launch.py pi 30000 720 > gpurun_out/r02y_ncu_pilanes.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nmpc_genw_kernel -s 1 -c 1 -o gpurun_out/r02y_k3w python tools/prof_launch.py nmpc3 1184 4 60 generic_warp > gpurun_out/r02y_ncu_k3w.log 2>&1
