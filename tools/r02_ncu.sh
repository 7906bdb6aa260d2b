mkdir -p gpurun_out
T=${TAG:-r02h}
timeout 120 python tools/train_exp.py shuffled > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_ws -s 2 -c 1 -o gpurun_out/${T}_train_ws python tools/train_exp.py shuffled > gpurun_out/${T}_ncu.log 2>&1
echo rc=$? >> gpurun_out/${T}_ncu.log
