set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02c2_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c2_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c2_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c2_smoke.txt
timeout 1500 python bench.py > gpurun_out/r02c2_bench_line.json 2> gpurun_out/r02c2_bench_err.txt; echo "rc=$?" >> gpurun_out/r02c2_bench_err.txt
