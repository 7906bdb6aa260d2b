# quick check of the warp-specialised train kernels
mkdir -p gpurun_out
T=${TAG:-r02c}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_divergence.py tests/test_gpu_stream.py tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in shuffled sorted; do for env in "" "NPM_DEBUG=1" "NPM_DEBUG=4" "NPM_BIN_TRAIN=1 NPM_PRIV_MAX=4096"; do env $env timeout 120 python tools/train_exp.py $v 2>&1 | grep -E "NPM_PHASES|variant" | tail -2 >> gpurun_out/${T}_exp.log; done; done
for w in c5 c3; do EXP_WORKLOAD=$w timeout 200 python tools/train_exp.py shuffled 2>&1 | tail -1 >> gpurun_out/${T}_exp.log; done
