mkdir -p gpurun_out
for lib in expt/k3_base.so expt/pi_div.so expt/k3_base.so expt/pi_div.so; do echo "== $lib"; NMPCMC_GPU_LIB=$PWD/$lib timeout 300 python tools/pi_time.py 5; done > gpurun_out/r02q_pi_div.txt 2>&1
python tools/ab_time.py 4736 10 60 expt/k3_base.so expt/pi_div.so expt/k3_base.so expt/pi_div.so > gpurun_out/r02q_k3_div.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_pi.py tests/test_gpu_nmpc.py tests/test_gpu_full.py tests/test_gpu_fuzz.py tests/test_gpu_units.py -m gpu -q -x > gpurun_out/r02q_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02q_pytest.txt
