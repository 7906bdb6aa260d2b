# same-box A/B of the query kernel: HEAD tree vs working tree vs ab/<v>.so
mkdir -p gpurun_out
T=${TAG:-r02qab}
O=gpurun_out/${T}_exp.log
: > $O
if [ -n "$TESTS" ]; then timeout 400 python -m pytest $TESTS -q -x --timeout 300 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log; fi
for i in 1 2; do
  echo -n "head " >> $O; (cd ab/headtree && timeout 150 python tools/query_exp.py 2>&1 | tail -1) >> $O
  echo -n "wt " >> $O; timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O
  for v in $VARIANTS; do echo -n "$v " >> $O; NPM_LIB=$PWD/ab/$v.so timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O; done
done
echo done
