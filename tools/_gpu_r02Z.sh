set -x
mkdir -p gpurun_out
timeout 2400 python tools/ab_time.py 9472 20 60 expt/b12.so expt/b12_qp2.so expt/b12_sh2.so expt/b12_sw2.so expt/b12_ro2.so expt/b12.so > gpurun_out/r02Z_k3_unroll_at12_ab.txt 2>&1
