# same-box A/B of libnpm variants on the training kernel (train_exp.py)
mkdir -p gpurun_out
O=gpurun_out/${TAG:-ab}_ab.log
: > $O
for i in 1 2; do for v in $VARIANTS; do for order in shuffled sorted; do
  echo -n "$v $order " >> $O
  NPM_LIB=$PWD/ab/$v.so timeout 120 python tools/train_exp.py $order 2>&1 | tail -1 >> $O
done; done; done
echo -n "r01kernel shuffled " >> $O; NPM_LIB=$PWD/ab/cur.so NPM_TRAIN_WS=0 timeout 120 python tools/train_exp.py shuffled 2>&1 | tail -1 >> $O
