# binning passes with batched loads: GPU tests, then same-box A/B (ab/head.so
# = HEAD, working tree) of the bench step at c2 / c3 / c5
mkdir -p gpurun_out
T=${TAG:-r02bin}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in head wt; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    for w in c2 c3 c5; do
      echo -n "$v $w " >> $O
      env $L timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O
    done
  done
done
echo done
