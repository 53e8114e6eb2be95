# ncu --set full capture of the count kernel for one configuration.
# usage: TAG=name bash tools/gpu_ncu.sh [env K=V ...]
mkdir -p gpurun_out
CMD="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-large ${BENCH_ARGS:-}"
env "$@" $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:count_ -s 12 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_${TAG}.log
