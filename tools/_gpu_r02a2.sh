set -x
mkdir -p gpurun_out
timeout 300 python tools/prof_launch.py nmpc 1776 6 60 > gpurun_out/r02a2_prof_plain.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nmpc_kernel -s 1 -c 1 -o gpurun_out/r02a2_k3 python tools/prof_launch.py nmpc 1776 6 60 > gpurun_out/r02a2_ncu_full.log 2>&1
timeout 900 python tools/ocp_bench.py 20000 60 > gpurun_out/r02a2_ocp_one_state.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_ocp.py tests/test_sqp_trace.py -m gpu -q > gpurun_out/r02a2_pytest_ocp.txt 2>&1; echo "rc=$?" >> gpurun_out/r02a2_pytest_ocp.txt
