# c5 query variants (ab/<v>.so) vs the working tree, same box; c5 parity on each
mkdir -p gpurun_out
T=${TAG:-r02c5q}
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in wt $VARIANTS; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    echo -n "$v c5 " >> $O; env $L EXP_WORKLOAD=c5 timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O
  done
done
for v in $VARIANTS; do
  NPM_LIB=$PWD/ab/$v.so timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "c5 and query" > gpurun_out/${T}_${v}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_${v}_pytest.log
done
echo done
