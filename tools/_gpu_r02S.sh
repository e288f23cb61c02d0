set -x
mkdir -p gpurun_out
{
timeout 1500 python tools/ab_time.py 9472 20 60 expt/fin.so expt/cg.so expt/fin.so expt/cg.so
for lib in expt/fin.so expt/cg.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 9472 10 60 0 generic_warp
done
} > gpurun_out/r02S_dlcm_cg_ab.txt 2>&1
