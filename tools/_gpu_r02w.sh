mkdir -p gpurun_out
{
for lib in expt/k3w_m3.so expt/k3w_tr.so expt/k3w_m3.so expt/k3w_tr.so; do
  echo "== $lib"
  NMPCMC_GPU_LIB=$PWD/$lib timeout 300 python tools/gen_time.py 2368 10 60 0 generic_warp
done
} > gpurun_out/r02w_k3w_ab.txt 2>&1
timeout 1500 python -m pytest tests/test_sqp_trace.py tests/test_gpu_ocp.py tests/test_gpu_gen.py tests/test_qnlp.py tests/test_controllers.py tests/test_gpu_fuzz.py -m gpu -q > gpurun_out/r02w_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02w_pytest.txt
