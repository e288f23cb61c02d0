set -x
mkdir -p gpurun_out
timeout 2400 python tools/ab_time.py 9472 20 60 expt/fin.so expt/k3_r144.so expt/k3_r152.so expt/k3_mb12.so expt/k3_r184.so expt/fin.so > gpurun_out/r02V_k3_regs_ab.txt 2>&1
