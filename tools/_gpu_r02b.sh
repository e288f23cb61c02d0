set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_integration.py tests/test_cpp_facade.py tests/test_gpu_nmpc.py tests/test_gpu_full.py -m gpu -q -x > gpurun_out/r02b_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02b_pytest.txt
timeout 300 python tools/prof_launch.py nmpc 2368 6 60 > gpurun_out/r02b_prof_plain.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nmpc_kernel -s 1 -c 1 -o gpurun_out/r02b_k3 python tools/prof_launch.py nmpc 2368 6 60 > gpurun_out/r02b_ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_ncu.csv python bench.py --steps 1 --warmup 3 --no-legs --no-cpu-baseline > gpurun_out/r02b_ncu_launch.log 2>&1
