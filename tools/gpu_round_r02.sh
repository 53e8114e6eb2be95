# Round-2 evidence (one gpurun call): GPU test suite, default bench line,
# reference arm, ncu launch list of the plain bench command, one ncu --set
# full capture of the count kernel at C4 and at C5.  Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/r02_gpu_tests.log
python bench.py > gpurun_out/r02_bench.log 2>&1; echo "EXIT $?" >> gpurun_out/r02_bench.log
python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r02_bench_ref.log 2>&1
CMD="python bench.py --steps 40 --warmup 3 --no-cpu-baseline --no-large"
$CMD > gpurun_out/r02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/r02_launches_c4.csv $CMD > gpurun_out/r02_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:count_ -s 12 -c 1 -o gpurun_out/prof_r02_c4_final $CMD > gpurun_out/r02_ncu_c4.log 2>&1
CMD5="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-large --workload c5"
$CMD5 > gpurun_out/r02_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_ -s 12 -c 1 -o gpurun_out/prof_r02_c5_final $CMD5 > gpurun_out/r02_ncu_c5.log 2>&1
echo done
