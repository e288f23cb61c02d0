set -x
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nmpc_genw_kernel -s 1 -c 1 -o gpurun_out/r02E_k3w python tools/prof_launch.py nmpc3 1184 3 60 generic_warp > gpurun_out/r02E_ncu.log 2>&1
