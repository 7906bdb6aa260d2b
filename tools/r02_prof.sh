# evidence run: plain bench (must exit 0), then the ncu launch list of the same
# command and one --set full capture per hot kernel (all ncu in one call)
mkdir -p gpurun_out
T=${TAG:-r02r}
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strong > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strong > gpurun_out/${T}_ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_ws -s 2 -c 1 -o gpurun_out/${T}_train_ws python tools/train_exp.py shuffled > gpurun_out/${T}_ncu_train.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_query -s 3 -c 1 -o gpurun_out/${T}_query python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-strong > gpurun_out/${T}_ncu_query.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_ncu_query.log
