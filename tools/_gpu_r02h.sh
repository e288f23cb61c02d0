mkdir -p gpurun_out
python tools/ab_time.py 4736 10 60 paper_2212_02197_b200/_lib/libnmpcmc_gpu.so expt/u_112/libnmpcmc_gpu.so expt/u_114/libnmpcmc_gpu.so expt/u_122/libnmpcmc_gpu.so expt/u_222/libnmpcmc_gpu.so paper_2212_02197_b200/_lib/libnmpcmc_gpu.so > gpurun_out/r02h_unroll_ab.txt 2>&1
