import sys, numpy as np
sys.path.insert(0, '.')
import paper_2512_04556_b200 as skc
from paper_2512_04556_b200 import synth
n = 16
tg = [synth.c4_target(i) for i in range(n)]
inits = [synth.c4_init(i) for i in range(n)]
for steps in (300, 1000, 3000):
    res = skc.fit_batch(tg, (32,)*4, inits, skc.TrainConfig(steps=steps), skc.ConstraintConfig("sum"), skc.LossKind("l1"))
    tot = []
    for r in res:
        c = r.canvas
        half = c // 2
        lo = hi = 0
        sizes = []
        for lay in r.complex.layers:
            fl = np.floor(lay.offsets)
            lo_x, hi_x = fl.min(), fl.max() + 1
            lo += -lo_x; hi += hi_x
            w = min(c, int(1 + lo + hi))
            sizes.append(w)
        tot.append(sum(s*s for s in sizes))
        if r is res[0]: print(steps, 'canvas', c, 'box widths', sizes, 'loss', r.final_loss)
    print(steps, 'sum box area mean/max', np.mean(tot), np.max(tot), 'arena floats', 47000)
