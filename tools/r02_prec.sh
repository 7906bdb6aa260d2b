# backward-MMA precision variants: gradient error vs the oracle, the parity and
# stream tests, and a same-box A/B of the training kernel (ab/<v>.so)
mkdir -p gpurun_out
T=${TAG:-r02prec}
O=gpurun_out/${T}_exp.log
: > $O
for v in wt $VARIANTS; do
  L=""; [ "$v" != wt ] && L="NPM_LIB=$PWD/ab/$v.so"
  echo -n "$v err " >> $O; env $L timeout 300 python tools/grad_err.py 2>&1 | tail -1 >> $O
  env $L timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x --timeout 300 2>&1 | tail -2 | sed "s/^/$v tests /" >> $O
done
for i in 1 2; do
  for v in wt $VARIANTS; do
    L=""; [ "$v" != wt ] && L="NPM_LIB=$PWD/ab/$v.so"
    echo -n "$v " >> $O; env $L timeout 300 python tools/train_exp.py shuffled 2>&1 | tail -1 >> $O
  done
done
echo done
