mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "rc=$?" >> gpurun_out/r02i_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02i_bench_ref.json 2> gpurun_out/r02i_bench_ref.err
