# c4 query without the unused hidden-buffer gap (ab/pnogap.so) vs the working tree
mkdir -p gpurun_out
T=${TAG:-r02pgap}
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in wt pnogap; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    echo -n "$v c4 " >> $O; env $L EXP_WORKLOAD=c4 timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O
  done
done
NPM_LIB=$PWD/ab/pnogap.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k c4 > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
echo done
