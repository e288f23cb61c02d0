set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py tests/test_gpu_ocp.py tests/test_qnlp.py tests/test_controllers.py tests/test_gpu_full.py tests/test_cli.py -m gpu -q -x > gpurun_out/r02L_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02L_pytest.txt
NMPCMC_GPU_LIB=$PWD/paper_2212_02197_b200/_lib/libnmpcmc_gpu.so timeout 600 python tools/gen_time.py 9472 10 60 0 generic_warp > gpurun_out/r02L_k3w_time.txt 2>&1
