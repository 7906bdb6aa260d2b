set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r01d_bench.json 2> gpurun_out/r01d_bench.err
for w in c3 c4 c5; do python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01d_bench_$w.json 2>/dev/null; done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01d_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tc_(train64|query)" -s 2 -c 2 -o gpurun_out/r01d_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r01d_ncu_full.log 2>&1
echo done
