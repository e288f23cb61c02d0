set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py 9472 20 60 expt/fin.so expt/k3_mb13.so expt/k3_mb12.so expt/fin.so > gpurun_out/r02T_k3_minblocks_ab.txt 2>&1
