set -x
mkdir -p gpurun_out
timeout 2400 python tools/ab_time.py 9472 20 60 expt/k3_mb12.so expt/k3_alias.so expt/k3_mb12.so expt/k3_alias.so > gpurun_out/r02X_k3_tmp_alias_ab.txt 2>&1
