# The bench line on BASELINE configs 1 and 3 (and the reference arm on C1), for profiles/.
mkdir -p gpurun_out
python bench.py --workload c1 > gpurun_out/r02_bench_c1.log 2>&1
python bench.py --impl reference --workload c1 --steps 20 --warmup 3 > gpurun_out/r02_bench_ref_c1.log 2>&1
python bench.py --workload c3 > gpurun_out/r02_bench_c3.log 2>&1
echo done
