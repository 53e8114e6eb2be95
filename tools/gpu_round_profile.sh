# Round evidence: full bench (default flags), reference arm, launch list and one
# ncu --set full capture of the count kernel.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "EXIT $?" >> gpurun_out/bench_full.log
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-large"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_tma -s 12 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_full.log
