"""Quick device timing of one closed-loop batch (dev tool, not the bench)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_02197_b200 import configs, engine, abi

def main():
    ctl = sys.argv[1] if len(sys.argv) > 1 else "pi"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
    kw = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
    sc = configs.make_scenario(ctl, perturb=True, **kw)
    ctx = engine.Context(0)
    ctx.set_nmpc_kernel(os.environ.get('KERNEL', 'warp'))
    if 'WPS' in os.environ: ctx.set_tps_warps_per_sm(int(os.environ['WPS']))
    rec = torch.empty(n * 24, dtype=torch.uint8, device="cuda")
    cnt = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    for it in range(int(os.environ.get("ITERS", "4"))):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        ctx.run_device(sc, 0, n, rec.data_ptr(), cnt.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
        c = np.frombuffer(cnt.cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE)
        print(f"{ctl} n={n} iter {it}: {ms:.3f} ms -> {n/ms*1e3:.1f} sims/s; failed {int(r['failed'].sum())}; "
              f"mean phi {np.nanmean(r['phi']):.4f}; counters {dict((k, int(c[k].sum())) for k in c.dtype.names)}", flush=True)

if __name__ == "__main__":
    main()
