# Round evidence, part 2: one `ncu --set full` capture of the count kernel on
# C4 (after the same command ran clean without ncu).  Output gpurun_out/prof_c4.ncu-rep.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-large"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_tma -s 12 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_full.log
