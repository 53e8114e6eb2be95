# Kernel-configuration sweep on the C4 workload (bench.py, no CPU baseline).
# usage: bash tools/gpu_sweep.sh "<env1>" "<env2>" ...   (each "K=V K2=V2")
mkdir -p gpurun_out
out=gpurun_out/sweep.log
: > $out
for cfg in "$@"; do
  echo "== $cfg" >> $out
  env $cfg timeout 300 python bench.py --steps 400 --warmup 5 --no-cpu-baseline --no-large ${BENCH_ARGS:-} 2>&1 | \
    python -c "import sys,json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline'] or {}
        print('value %.3e  us/launch %.2f  frac %.3f  e2e %.3e  pyapi %s b2b_us %.2f phases %s cfg %s' % (d['value'], r.get('avg_launch_us') or 0, r.get('frac') or 0, (d['e2e'] or {}).get('value') or 0, (d.get('e2e_python_api') or {}).get('value'), d.get('diag_back_to_back_us_per_step') or 0, d.get('phases'), d['kernel_config']))
    else: print(l[:300])" >> $out
done
