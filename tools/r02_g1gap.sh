# GPU tests of the working tree; c5 query with the one-group gap dropped
# (ab/g1nogap.so) vs the working tree
mkdir -p gpurun_out
T=${TAG:-r02g1gap}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in wt g1nogap; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    for w in c4 c5; do echo -n "$v $w " >> $O; env $L EXP_WORKLOAD=$w timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O; done
  done
done
echo done
