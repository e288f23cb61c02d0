set -x
mkdir -p gpurun_out
timeout 2400 python tools/sweep_config4.py --sims 10000 100000 --horizons 30 60 120 > gpurun_out/r02e2_cfg4_sweep.jsonl 2> gpurun_out/r02e2_cfg4_sweep.err
