set -x
mkdir -p gpurun_out
L=$PWD/paper_2212_02197_b200/_lib/libnmpcmc_gpu.so
{
echo "== L2 persist off"; timeout 600 python tools/ab_time.py 9472 20 60 $L
echo "== L2 persist on"; NMPCMC_L2_PERSIST=1 timeout 600 python tools/ab_time.py 9472 20 60 $L
echo "== L2 persist off"; timeout 600 python tools/ab_time.py 2368 20 60 $L
echo "== L2 persist on"; NMPCMC_L2_PERSIST=1 timeout 600 python tools/ab_time.py 2368 20 60 $L
} > gpurun_out/r02H_l2persist_ab.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:nmpc_kernel -s 1 -c 1 --csv --log-file gpurun_out/r02H_dram_off.csv python tools/prof_launch.py nmpc 2368 6 60 > gpurun_out/r02H_off.log 2>&1
NMPCMC_L2_PERSIST=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:nmpc_kernel -s 1 -c 1 --csv --log-file gpurun_out/r02H_dram_on.csv python tools/prof_launch.py nmpc 2368 6 60 > gpurun_out/r02H_on.log 2>&1
