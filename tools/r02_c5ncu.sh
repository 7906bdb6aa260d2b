# c5 (HBM-resident tables) at HEAD: query (one chain group) and train kernel
# ncu --set full, each after the same command exited 0 without ncu
mkdir -p gpurun_out
T=${TAG:-r02c5}
EXP_WORKLOAD=c5 timeout 300 python tools/query_exp.py > gpurun_out/${T}_query_plain.log 2>&1 && \
EXP_WORKLOAD=c5 timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_ws -s 3 -c 1 -o gpurun_out/${T}_query_ws python tools/query_exp.py > gpurun_out/${T}_ncu_query.log 2>&1
echo "ncu query rc=$?" >> gpurun_out/${T}_ncu_query.log
EXP_WORKLOAD=c5 timeout 300 python tools/train_exp.py shuffled > gpurun_out/${T}_train_plain.log 2>&1 && \
EXP_WORKLOAD=c5 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_train64 -s 2 -c 1 -o gpurun_out/${T}_train64 python tools/train_exp.py shuffled > gpurun_out/${T}_ncu_train.log 2>&1
echo "ncu train rc=$?" >> gpurun_out/${T}_ncu_train.log
echo done
