set -x
mkdir -p gpurun_out
for lib in expt/k3w_prev.so paper_2212_02197_b200/_lib/libnmpcmc_gpu.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 2368 10 60 0 generic_warp
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 9472 10 60 0 generic_warp
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 9472 10 60 1 generic_warp
done > gpurun_out/r02M_k3w_ab.txt 2>&1
