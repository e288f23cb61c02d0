set -x
mkdir -p gpurun_out
for lib in expt/k3w_noqq.so expt/k3w_nj.so expt/k3w_nj224.so expt/k3w_nj200.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 2368 10 60 0 generic_warp
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 9472 10 60 0 generic_warp
done > gpurun_out/r02K_k3w_ab.txt 2>&1
