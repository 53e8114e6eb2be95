python -m pytest tests/test_gpu_parity.py -x -q -k "compact or c5 or wide or dirty or edge" > gpurun_out/pytest_compact.log 2>&1; tail -15 gpurun_out/pytest_compact.log
BENCH_ARGS="--workload c5" bash tools/gpu_sweep.sh "EBIC_COMPACT=0" "EBIC_COMPACT=-1" "EBIC_COMPACT=1 EBIC_SLICE=64" "EBIC_COMPACT=1 EBIC_SLICE=64 EBIC_NCW=16"
cat gpurun_out/sweep.log
