set -x
mkdir -p gpurun_out
{
timeout 1500 python tools/ab_time.py 9472 20 60 expt/cur.so expt/pair.so expt/cur.so expt/pair.so
echo "== N=120"; timeout 1200 python tools/ab_time.py 4736 20 120 expt/cur.so expt/pair.so
echo "== N=40"; timeout 1200 python tools/ab_time.py 9472 20 40 expt/cur.so expt/pair.so
} > gpurun_out/r02d2_k3_shoot_pair_ab.txt 2>&1
