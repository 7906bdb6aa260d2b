# same-box A/B incl. binned training (NPM_BIN_TRAIN=1 with / without privatised coarse levels)
mkdir -p gpurun_out
O=gpurun_out/${TAG:-ab}_ab.log
: > $O
for v in $VARIANTS; do for order in shuffled sorted; do for env in "" "NPM_BIN_TRAIN=1 NPM_PRIV=0" "NPM_BIN_TRAIN=1 NPM_PRIV_MAX=4096"; do
  echo -n "$v $order [$env] " >> $O
  env $env NPM_LIB=$PWD/ab/$v.so timeout 120 python tools/train_exp.py $order 2>&1 | tail -1 >> $O
done; done; done
