# compute-sanitizer memcheck over the generated sparse stencils (fp32 / fp16, heads, planar and HWC epilogues, ragged sizes)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2512_04556_b200 as skc
from paper_2512_04556_b200 import synth
rng = np.random.default_rng(1)
for cpx in (synth.c1_complex(), synth.c0_complex()):
    for shape in ((131, 97, 3), (61, 300, 1), (200, 129, 4)):
        for dt in (np.float32, np.float16):
            x = rng.random(shape).astype(dt)
            for mode in ("zero", "clamp"):
                skc.apply_complex(x, cpx, boundary=mode)
kaw = synth.kawase_complex()
for shape in ((99, 131, 4), (40, 37, 4)):
    x = rng.random(shape).astype(np.float16)
    for mode in ("zero", "clamp"):
        skc.apply_complex(x, kaw, boundary=mode)
basis = synth.c2_basis()
img = rng.random((150, 170, 3)).astype(np.float32)
skc.sv_filter(img, basis, synth.c2_pmap(150, 170, seed=5, blobs=4))
print("done")
PY
python /tmp/san.py > /dev/null 2>&1   # warm the kernel cache outside the sanitizer
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > gpurun_out/sanitizer90.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/sanitizer90.log
