#!/bin/bash
# round 2: Kawase kernel parity + timing
set -x
export SKC_CACHE_DIR=$(mktemp -d)
timeout 600 python -m pytest tests/test_gpu_kawase.py -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/kw_test.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/kw_bench_c3.json 2> gpurun_out/kw_bench_c3.err
timeout 300 python bench.py --config c3big --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/kw_bench_c3big.json 2> gpurun_out/kw_bench_c3big.err
