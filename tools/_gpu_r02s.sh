mkdir -p gpurun_out
{
for lib in expt/k3w_m0.so expt/k3w_m1/libnmpcmc_gpu.so expt/k3w_m0.so expt/k3w_m1/libnmpcmc_gpu.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 300 python tools/gen_time.py 2368 10 60 0 generic_warp
  NMPCMC_GPU_LIB=$PWD/$lib timeout 300 python tools/gen_time.py 2368 10 60 1 generic_warp
done
} > gpurun_out/r02s_k3w_model_ab.txt 2>&1
