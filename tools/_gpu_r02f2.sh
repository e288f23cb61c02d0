set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py 9472 20 120 expt/cur.so expt/nc.so expt/cur.so expt/nc.so > gpurun_out/r02f2_k3_n120_cert_ab.txt 2>&1
