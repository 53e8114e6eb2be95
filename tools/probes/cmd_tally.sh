timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_tally.log 2>&1; tail -3 gpurun_out/pytest_tally.log
bash tools/gpu_sweep.sh "EBIC_NCW=24" "EBIC_SPG=4" "EBIC_NCW=16"; cat gpurun_out/sweep.log
BENCH_ARGS="--workload c5" bash tools/gpu_sweep.sh "EBIC_NCW=24" "EBIC_NCW=31"; cat gpurun_out/sweep.log
