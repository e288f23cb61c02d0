"""Device time of the PI closed-loop kernel (K2) on BASELINE configs 0 and 1:
best of R launches, CUDA events on the context stream.

  python tools/pi_time.py [reps] [kernels]   (kernels: comma list of
  auto,lanes,ws3,ws7; default auto)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2212_02197_b200 import configs, engine, workmodel

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
kernels = sys.argv[2].split(",") if len(sys.argv) > 2 else ["auto"]
ctx = engine.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
for kern, (name, kw, n) in [(k, c) for k in kernels for c in (("config0", dict(controller="pi"), 1000), ("config1", dict(controller="pi", perturb=True), 30000),
                    ("config1_x4", dict(controller="pi", perturb=True), 120000))]:
    ctx.set_pi_kernel(kern)
    sc = configs.make_scenario(**kw)
    rec = torch.empty(n * 24, dtype=torch.uint8, device="cuda")
    cnt = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
    best = 1e9
    for r in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.run_device(sc, 0, n, rec.data_ptr(), cnt.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            best = min(best, e0.elapsed_time(e1))
    import numpy as np
    from paper_2212_02197_b200 import abi
    c = np.frombuffer(cnt.cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE)
    fl = workmodel.pi_flops(int(c["control_steps"].sum()))
    import hashlib
    h = hashlib.sha1(rec.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"PI[{kern}] {name}: {n} sims, {best:.3f} ms, {n / best * 1e3:.0f} sims/s, {fl / best / 1e9:.3f} TF/s, rec {h}")
