# variance-aware target: own-part lobe pairs once each (ab/vasym.so) vs the working tree
mkdir -p gpurun_out
T=${TAG:-r02va}
O=gpurun_out/${T}_exp.log
: > $O
NPM_LIB=$PWD/ab/vasym.so timeout 600 python -m pytest tests/test_gpu_variance.py -q -x > gpurun_out/${T}_vasym_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_vasym_pytest.log
for i in 1 2; do
  for v in wt vasym; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    echo -n "$v " >> $O; env $L timeout 300 python tools/train_exp.py va 2>&1 | tail -1 >> $O
  done
done
echo done
