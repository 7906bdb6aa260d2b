mkdir -p gpurun_out
T=${TAG:-r02f}
for v in shuffled sorted; do for env in "NPM_DEBUG=4" "NPM_DEBUG=5"; do env $env timeout 120 python tools/train_exp.py $v 2>&1 | grep -E "NPM_PHASES|variant" | tail -2 >> gpurun_out/${T}_phase.log; done; done
