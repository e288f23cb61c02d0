set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02g2_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02g2_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g2_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r02g2_smoke.txt
{
echo "== N=120"; timeout 1500 python tools/ab_time.py 9472 20 120 expt/cur.so expt/new.so
echo "== N=200"; timeout 1500 python tools/ab_time.py 2368 10 200 expt/cur.so expt/new.so
echo "== N=60"; timeout 1500 python tools/ab_time.py 9472 20 60 expt/cur.so expt/new.so
} > gpurun_out/r02g2_k3_cert_per_stride_ab.txt 2>&1
timeout 1500 python tools/sweep_config4.py --sims 10000 100000 --horizons 120 > gpurun_out/r02g2_cfg4_n120.jsonl 2> gpurun_out/r02g2_cfg4_n120.err
