set -x
mkdir -p gpurun_out
timeout 2400 python tools/ab_time.py 9472 20 60 expt/k3_mb12.so expt/k3_mb12ipm.so expt/k3_mb12nc.so expt/k3_mb12.so > gpurun_out/r02W_k3_mb12_variants_ab.txt 2>&1
NMPCMC_GPU_LIB=$PWD/expt/k3_mb12.so timeout 1200 python bench.py --steps 3 --warmup 3 --no-legs --no-cpu-baseline > gpurun_out/r02W_bench_mb12.json 2> gpurun_out/r02W_bench_mb12.err
NMPCMC_GPU_LIB=$PWD/expt/fin.so timeout 1200 python bench.py --steps 3 --warmup 3 --no-legs --no-cpu-baseline > gpurun_out/r02W_bench_fin.json 2> gpurun_out/r02W_bench_fin.err
