# fit FFMA2 (column pairs) A/B, library variants swapped in place
mkdir -p gpurun_out
cd paper_2512_04556_b200
cp libskc_f2.so libskc.so
(cd .. && python -m pytest tests/test_gpu_sv_fit.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log)
for v in f2 f0 f2 f0; do
  cp libskc_$v.so libskc.so
  (cd .. && python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b53_$v.json 2> gpurun_out/b53.err; echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/b53_$v.json').read().strip().splitlines()[-1]);print(d['value'])")")
done
