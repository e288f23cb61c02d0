set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py 9472 20 60 expt/k3_base2.so expt/k3_shexp.so expt/k3_base2.so expt/k3_shexp.so > gpurun_out/r02P_k3_shared_expand_ab.txt 2>&1
