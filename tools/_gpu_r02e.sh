mkdir -p gpurun_out
timeout 300 python tools/pi_time.py 5 > gpurun_out/r02e_pi_time.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02e_pytest.txt
