set -x
mkdir -p gpurun_out
timeout 2000 python tools/ab_time.py 9472 20 60 expt/fin.so expt/k3_mb12.so expt/k3_mb11.so expt/k3_mb10.so expt/k3_mb8.so > gpurun_out/r02U_k3_minblocks_ab.txt 2>&1
timeout 2000 python tools/ab_time.py 18944 20 60 expt/fin.so expt/k3_mb12.so expt/k3_mb10.so >> gpurun_out/r02U_k3_minblocks_ab.txt 2>&1
