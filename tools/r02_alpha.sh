# f-4' GPU check: alpha tests + the parity suites they share helpers with, and
# the training kernel's cost with / without the selection head
mkdir -p gpurun_out
T=${TAG:-r02al}
timeout 900 python -m pytest tests/test_gpu_alpha.py tests/test_gpu_parity.py tests/test_gpu_guide.py -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for v in ${VARIANTS:-shuffled alpha shuffled alpha}; do timeout 300 python tools/train_exp.py $v >> gpurun_out/${T}_exp.log 2>&1; done
echo done
