timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/probes/e2e_run.py c4 "EBIC_GRAPH=0" "EBIC_GRAPH=1" "EBIC_GRAPH=0" "EBIC_GRAPH=1" 2>&1 | grep -o "\['.*us_per_step\": [0-9.]*\|host_us.*}}"
bash tools/gpu_sweep.sh "EBIC_GRAPH=0" "EBIC_GRAPH=1"; cat gpurun_out/sweep.log
