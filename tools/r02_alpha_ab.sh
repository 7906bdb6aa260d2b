# f-4' check: alpha parity tests, then same-box A/B of the training kernel:
# HEAD tree (ab/headtree, built there) vs the working tree (plain, learn_alpha,
# and measurement variants ab/<v>.so)
mkdir -p gpurun_out
T=${TAG:-r02ab}
timeout 900 python -m pytest tests/test_gpu_alpha.py tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  echo -n "head " >> $O; (cd ab/headtree && timeout 300 python tools/train_exp.py shuffled 2>&1 | tail -1) >> $O
  echo -n "wt " >> $O; timeout 300 python tools/train_exp.py shuffled 2>&1 | tail -1 >> $O
  echo -n "wt " >> $O; timeout 300 python tools/train_exp.py alpha 2>&1 | tail -1 >> $O
  for v in $VARIANTS; do echo -n "$v " >> $O; NPM_LIB=$PWD/ab/$v.so timeout 300 python tools/train_exp.py shuffled 2>&1 | tail -1 >> $O; done
done
echo done
