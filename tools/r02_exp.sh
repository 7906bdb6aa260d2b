# train-kernel knob experiment at c2 (measurement only)
mkdir -p gpurun_out
O=gpurun_out/${TAG:-r02b}_exp.log
: > $O
for v in shuffled sorted; do
  for env in "" "NPM_DEBUG=1" "NPM_BIN_TRAIN=1" "NPM_BIN_TRAIN=1 NPM_PRIV=0" "NPM_BIN_TRAIN=1 NPM_DEBUG=1" "NPM_DEBUG=8" "NPM_DEBUG=16"; do
    env $env timeout 120 python tools/train_exp.py $v >> $O 2>&1
  done
done
echo done >> $O
