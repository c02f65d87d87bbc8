# fit: loss-loop unroll A/B (library variants swapped in place)
mkdir -p gpurun_out
cd paper_2512_04556_b200
for v in unroll nounroll unroll nounroll; do
  cp libskc_$v.so libskc.so
  (cd .. && python bench.py --config c4 --no-e2e --no-cpu > gpurun_out/b44_$v.json 2> gpurun_out/b44.err; echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/b44_$v.json').read().strip().splitlines()[-1]);print(d['value'])")")
done
