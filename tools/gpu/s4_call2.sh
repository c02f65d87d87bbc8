# session 4: Kawase H warm-up peel A/B, Kawase parity, ncu capture; PCIe duplex probe; c0 fused
mkdir -p gpurun_out/s4b
export SKC_CACHE_DIR=$(mktemp -d)
show() { python -c "
import json,sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'per', [round(t,3) for t in d['roofline'].get('per_launch_ms', [])])
" $1; }
for v in 1 0 1 0; do
  SKC_KAWASE_PEEL=$v timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4b/c3_peel$v.json 2> gpurun_out/s4b/c3_peel$v.err; echo "c3 peel=$v rc=$?"; show gpurun_out/s4b/c3_peel$v.json
done
timeout 300 python bench.py --config c3big --steps 10 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4b/c3big.json 2>&1; show gpurun_out/s4b/c3big.json
timeout 900 python -m pytest tests/test_gpu_kawase.py -m gpu -q -p no:cacheprovider > gpurun_out/s4b/kawase_tests.log 2>&1; echo "kawase tests rc=$?"; tail -2 gpurun_out/s4b/kawase_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kawase_sep -c 1 -o gpurun_out/s4b/kawase_peel python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-others > gpurun_out/s4b/ncu_kw.log 2>&1; echo "ncu rc=$?"
SKC_FUSED=1 timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4b/c0_fused.json 2>&1; show gpurun_out/s4b/c0_fused.json
timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-e2e --no-cpu --no-others > gpurun_out/s4b/c0.json 2>&1; show gpurun_out/s4b/c0.json
python - <<'PY'
import torch, time
n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device='cuda'); d_b = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return n * reps / dt / 1e9
run(True, True, 2)
print('h2d only GB/s', round(run(True, False), 1), 'd2h only', round(run(False, True), 1), 'duplex per direction', round(run(True, True), 1))
PY
