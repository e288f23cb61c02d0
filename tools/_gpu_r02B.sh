set -x
mkdir -p gpurun_out
timeout 1200 python tools/ab_time.py 2368 20 60 expt/base.so expt/w1.so expt/w4.so expt/w8.so expt/w16.so > gpurun_out/r02B_ab_2368x20.txt 2>&1
timeout 1200 python tools/ab_time.py 9472 40 60 expt/base.so expt/w1.so expt/w4.so expt/w16.so > gpurun_out/r02B_ab_9472x40.txt 2>&1
