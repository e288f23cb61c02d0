mkdir -p gpurun_out
python tools/ab_time.py 4736 10 60 expt/k3_base.so expt/k3_cert/libnmpcmc_gpu.so expt/k3_base.so expt/k3_cert/libnmpcmc_gpu.so expt/k3_base.so expt/k3_cert/libnmpcmc_gpu.so > gpurun_out/r02o_k3_cert_ab.txt 2>&1
