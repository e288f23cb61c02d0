set -x
mkdir -p gpurun_out
{
echo "== N=30"; timeout 1200 python tools/ab_time.py 9472 20 30 expt/b16.so expt/b12.so
echo "== N=120"; timeout 1200 python tools/ab_time.py 4736 20 120 expt/b16.so expt/b12.so
echo "== N=60, 1000 samples (config 2 size)"; timeout 1200 python tools/ab_time.py 1000 40 60 expt/b16.so expt/b12.so
} > gpurun_out/r02b2_k3_minblocks_other_N.txt 2>&1
