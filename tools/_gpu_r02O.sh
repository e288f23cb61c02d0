set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_time.py 9472 20 60 expt/k3_base2.so expt/k3_qp2.so expt/k3_sh2.so expt/k3_base2.so > gpurun_out/r02O_k3_lane_unroll_ab.txt 2>&1
