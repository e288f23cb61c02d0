mkdir -p gpurun_out
for d in expt/pi_g*/; do echo "== $d"; NMPCMC_GPU_LIB=$PWD/$d/libnmpcmc_gpu.so timeout 300 python tools/pi_time.py 5; done > gpurun_out/r02c_pi_variants.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_pi.py tests/test_controllers.py tests/test_cli.py tests/test_cpp_facade.py tests/test_gpu_units.py -m gpu -q -x > gpurun_out/r02c_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c_pytest.txt
