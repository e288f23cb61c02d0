set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02Y_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02Y_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02Y_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02Y_smoke.txt
timeout 1500 python bench.py > gpurun_out/r02Y_bench_line.json 2> gpurun_out/r02Y_bench_err.txt; echo "rc=$?" >> gpurun_out/r02Y_bench_err.txt
timeout 900 python bench.py --impl reference > gpurun_out/r02Y_bench_ref_line.json 2> gpurun_out/r02Y_bench_ref_err.txt; echo "rc=$?" >> gpurun_out/r02Y_bench_ref_err.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02Y_launches_ncu.csv python bench.py --steps 1 --warmup 3 --no-legs --no-cpu-baseline > gpurun_out/r02Y_ncu_launch.log 2>&1
timeout 900 python tools/ocp_bench.py 20000 60 > gpurun_out/r02Y_ocp_one_state.txt 2>&1
