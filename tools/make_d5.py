"""SURVEY D5(iii) fixture: the config-4 fit statistic from the float64 oracle.

Runs all 256 config-4 targets (synth.c4_target / c4_init) for 3000 steps of
fit() -- TrainConfig(steps=3000) default schedule, SUM weights, L1 loss, the
same call bench.py's c4 workload makes -- through the pinned C oracle
(oracle/skc_oracle.c or_fit_batch, optim.py:390-469), twice: once from the
exact inits and once with every offset perturbed by a relative 1e-7 (seeded),
which measures the reference's own chaotic spread.

Writes tests/golden/d5_c4_fit.npz (final/best losses, canvas, the first 21
trace entries and every 100th).  TEST INFRASTRUCTURE: ~30 min per run on 8
host cores.  Usage: python tools/make_d5.py [--targets 256] [--steps 3000]
"""

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle as orc  # noqa: E402
from paper_2512_04556_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--targets", type=int, default=256)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "d5_c4_fit.npz"))
    a = ap.parse_args()
    if a.threads:
        orc.set_threads(a.threads)
    n = a.targets
    tg = np.stack([synth.c4_target(i).weights for i in range(n)])
    inits = [synth.c4_init(i) for i in range(n)]
    off0 = np.stack([np.concatenate([l.offsets for l in c.layers]) for c in inits]).astype(np.float64)
    w0 = np.stack([np.concatenate([l.weights for l in c.layers]) for c in inits]).astype(np.float64)
    rng = np.random.default_rng(12345)
    off_p = off0 * (1.0 + 1e-7 * rng.uniform(-1.0, 1.0, off0.shape))
    res = {}
    for tag, off in (("exact", off0), ("perturbed", off_p)):
        t0 = time.time()
        r = orc.fit_batch(tg, off, w0, [32] * 4, steps=a.steps, weight_norm="sum", loss_kind="l1")
        print(f"{tag}: {time.time() - t0:.0f}s, rc {np.unique(r['rc'])}, mean final "
              f"{r['trace'][:, -1].mean():.6f}", flush=True)
        res[tag] = r
    keep = np.arange(0, a.steps + 1, 100)
    out = {"targets": n, "steps": a.steps}
    for tag, r in res.items():
        out[f"{tag}_final"] = r["trace"][:, -1]
        out[f"{tag}_best"] = r["best_loss"]
        out[f"{tag}_best_step"] = r["best_step"]
        out[f"{tag}_canvas"] = r["canvas"]
        out[f"{tag}_rc"] = r["rc"]
        out[f"{tag}_early"] = r["trace"][:, :21]
        out[f"{tag}_every100"] = r["trace"][:, keep]
    np.savez_compressed(a.out, **out)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
