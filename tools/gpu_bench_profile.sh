set -x
python bench.py > gpurun_out/bench2.log 2>&1; echo EXIT $? >> gpurun_out/bench2.log
CMD="python bench.py --steps 60 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_tma -s 20 -c 2 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo NCU EXIT $? >> gpurun_out/ncu_full.log
