# HWC epilogue variants test (incl. the cluster-of-C epilogue)
mkdir -p gpurun_out
export SKC_CACHE_DIR=/tmp/skc_cache
python -m pytest tests/test_gpu_engine.py -m gpu -x -q -k "epilogue" > gpurun_out/pytest_gpu83.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu83.log
