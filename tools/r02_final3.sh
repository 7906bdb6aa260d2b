# round-2 final evidence on one box (+ the c4 training kernel): tests, smoke, bench (+reference, c3/c4/c5),
# then the ncu launch list and --set full captures of the two hot kernels, each
# directly after the same command exited 0 without ncu
set -x
mkdir -p gpurun_out
T=${TAG:-r02v5}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for w in c3 c4 c5; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-strong > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strong > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strong > gpurun_out/${T}_ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/${T}_ncu_launch.log
timeout 300 python tools/train_exp.py shuffled > gpurun_out/${T}_train_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_ws -s 2 -c 1 -o gpurun_out/${T}_train_ws python tools/train_exp.py shuffled > gpurun_out/${T}_ncu_train.log 2>&1
echo "ncu train rc=$?" >> gpurun_out/${T}_ncu_train.log
timeout 300 python tools/query_exp.py > gpurun_out/${T}_query_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_ws -s 3 -c 1 -o gpurun_out/${T}_query_ws python tools/query_exp.py > gpurun_out/${T}_ncu_query.log 2>&1
echo "ncu query rc=$?" >> gpurun_out/${T}_ncu_query.log
timeout 600 python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-strong > gpurun_out/${T}_c4_plain.json 2> gpurun_out/${T}_c4_plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_ws -s 2 -c 1 -o gpurun_out/${T}_c4_train_ws python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline --no-strong > gpurun_out/${T}_ncu_c4_train.log 2>&1
echo "ncu c4 train rc=$?" >> gpurun_out/${T}_ncu_c4_train.log
echo done
