"""Time a default-size parallel-tempering run on the device.

pst_fit with the reference's defaults (10 chains x 10 000 iterations, swap
every 10) on a 4 x 8 complex against a 33 x 33 disk target: every iteration
is proposals + 10 impulse responses + Metropolis + bookkeeping on the device
(skc_pst_run), one host sync at the start and one at the end.

    python tools/bench_pst.py [--iterations N] [--chains C]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iterations", type=int, default=10000)
    ap.add_argument("--chains", type=int, default=10)
    ap.add_argument("--layout", default="4x8")
    a = ap.parse_args()
    import torch
    import paper_2512_04556_b200 as skc
    tgt = skc.disk_kernel(12.0, 33)
    cfg = skc.PSTConfig(chains=a.chains, iterations=a.iterations, seed=1)
    skc.pst_fit(tgt, a.layout, skc.PSTConfig(chains=a.chains, iterations=64, seed=0), skc.InitStrategy("ss", seed=1),
                skc.LossKind("l1"))        # warm-up (graph capture, allocations)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = skc.pst_fit(tgt, a.layout, cfg, skc.InitStrategy("ss", seed=1), skc.LossKind("l1"))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"what": "pst_fit (device-resident)", "chains": a.chains, "iterations": a.iterations,
                      "layout": a.layout, "target": "disk r=12, 33x33", "seconds": dt,
                      "iterations_per_s": a.iterations / dt, "chain_energy_evals_per_s": a.iterations * a.chains / dt,
                      "best_energy": res.best_energy, "accept_rate": (res.accepts / a.iterations).tolist()}))


if __name__ == "__main__":
    main()
