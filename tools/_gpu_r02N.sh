set -x
mkdir -p gpurun_out
{
timeout 900 python tools/ocp_bench.py 20000 60 three
timeout 900 python tools/ocp_bench.py 20000 60
} > gpurun_out/r02N_ocp_service.txt 2>&1
