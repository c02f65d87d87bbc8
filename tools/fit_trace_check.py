"""Compare GPU fit traces with the float64 oracle step by step (diagnostic)."""
import sys, json, numpy as np
sys.path.insert(0, '.')
n, steps = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "both"
from paper_2512_04556_b200 import synth
tg = [synth.c4_target(i) for i in range(n)]
inits = [synth.c4_init(i) for i in range(n)]
if mode in ("oracle", "both"):
    from oracle import oracle as orc
    off0 = np.stack([np.concatenate([l.offsets for l in c.layers]) for c in inits])
    w0 = np.stack([np.concatenate([l.weights for l in c.layers]) for c in inits])
    ref = orc.fit_batch(np.stack([t.weights for t in tg]), off0, w0, [32]*4, steps=steps, weight_norm="sum", loss_kind="l1")
    np.save(f"/tmp/oracle_trace_{n}_{steps}.npy", ref["trace"])
if mode in ("gpu", "both"):
    import paper_2512_04556_b200 as skc
    res = skc.fit_batch(tg, (32,)*4, inits, skc.TrainConfig(steps=steps), skc.ConstraintConfig("sum"), skc.LossKind("l1"))
    gpu = np.stack([r.losses for r in res])
    np.save(f"gpurun_out/gpu_trace_{n}_{steps}.npy", gpu)
    print("gpu final", gpu[:, -1])
