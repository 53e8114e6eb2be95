# Round evidence, part 1 (one ncu pass per gpurun call):
#   full bench (default flags), reference arm, the ncu launch list of the
#   plain bench command, GA-side comparisons (full runs, top-rank replay).
# Part 2 is tools/gpu_ncu_full.sh.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "EXIT $?" >> gpurun_out/bench_full.log
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python tools/toprank_compare.py > gpurun_out/toprank_compare.log 2>&1
bash tools/ga_run_compare.sh > /dev/null 2>&1
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-large"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "NCU EXIT $?" >> gpurun_out/ncu_list.log
