# c4 query: one chain group (ab/pg1.so) vs two (working tree), same box; the
# c4 parity tests on the variant; tools/san_small.py on the working tree
mkdir -p gpurun_out
T=${TAG:-r02pg}
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in wt pg1; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    echo -n "$v c4 " >> $O; env $L EXP_WORKLOAD=c4 timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O
  done
done
NPM_LIB=$PWD/ab/pg1.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k c4 > gpurun_out/${T}_pg1_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pg1_pytest.log
timeout 600 python tools/san_small.py > gpurun_out/${T}_san_small.log 2>&1; echo rc=$? >> gpurun_out/${T}_san_small.log
echo done
