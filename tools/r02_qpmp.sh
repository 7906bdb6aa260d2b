# same-box A/B of the query kernel: HEAD build (ab/head.so) vs the working
# tree vs ab/<v>.so at c2 and c4, plus the bench's f-1 / f-2 timings at c2
mkdir -p gpurun_out
T=${TAG:-r02qpmp}
O=gpurun_out/${T}_exp.log
: > $O
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log; fi
lib() { [ "$1" = wt ] && echo X=1 || echo NPM_LIB=$PWD/ab/$1.so; }
for i in 1 2; do
  for v in head wt $VARIANTS; do
    for w in c2 c4; do echo -n "$v $w " >> $O; env $(lib $v) EXP_WORKLOAD=$w timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O; done
    echo -n "$v f1f2 " >> $O; env $(lib $v) timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('extras', d); print({k: v for k, v in d.items() if k.startswith('f1') or k.startswith('f2')})" >> $O
  done
done
echo done
