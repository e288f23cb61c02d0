mkdir -p gpurun_out
for lib in paper_2212_02197_b200/_lib/libnmpcmc_gpu.so expt/pi2_g2/libnmpcmc_gpu.so expt/pi2_g4/libnmpcmc_gpu.so paper_2212_02197_b200/_lib/libnmpcmc_gpu.so; do echo "== $lib"; NMPCMC_GPU_LIB=$PWD/$lib timeout 300 python tools/pi_time.py 5; done > gpurun_out/r02p_pi_lanes.txt 2>&1
