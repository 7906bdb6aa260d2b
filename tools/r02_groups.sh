# chain-group selection per model: GPU tests, then c2 / c4 / c5 bench lines
mkdir -p gpurun_out
T=${TAG:-r02grp}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for w in c2 c4 c5; do
  echo -n "$w " >> $O
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['value'], d['e2e']['value'], {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O
done
echo done
