mkdir -p gpurun_out
for S in 7500 10000 15000; do
  timeout 900 python bench.py --steps 2 --warmup 3 --sims-per-step $S --no-legs --no-cpu-baseline > gpurun_out/r02g_bench_S$S.json 2> gpurun_out/r02g_bench_S$S.err
done
