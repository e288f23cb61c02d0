set -x
mkdir -p gpurun_out
for lib in expt/split2.so paper_2212_02197_b200/_lib/libnmpcmc_gpu.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 2368 10 60 0 generic_warp
  NMPCMC_GPU_LIB=$PWD/$lib timeout 600 python tools/gen_time.py 9472 10 60 0 generic_warp
done > gpurun_out/r02G_k3w_ab.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py tests/test_gpu_ocp.py tests/test_qnlp.py tests/test_controllers.py -m gpu -q -x > gpurun_out/r02G_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02G_pytest.txt
