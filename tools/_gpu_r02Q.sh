set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiny_horizon.py -m gpu -q > gpurun_out/r02Q_pytest_tiny.txt 2>&1; echo "rc=$?" >> gpurun_out/r02Q_pytest_tiny.txt
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 7 python tools/gen_time.py 64 2 60 0 generic_warp > gpurun_out/r02Q_memcheck_k3w.txt 2>&1; echo "rc=$?" >> gpurun_out/r02Q_memcheck_k3w.txt
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests/test_gpu_tiny_horizon.py -m gpu -q > gpurun_out/r02Q_memcheck_tiny.txt 2>&1; echo "rc=$?" >> gpurun_out/r02Q_memcheck_tiny.txt
