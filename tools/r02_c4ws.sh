# product shape in the warp-specialised training kernel: GPU tests, then a
# same-box A/B of c4 (default ws vs NPM_TRAIN_WS=0, the r01 kernel)
mkdir -p gpurun_out
T=${TAG:-r02c4}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in 1 0; do
    echo -n "ws=$v " >> $O
    NPM_TRAIN_WS=$v timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['value'], {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O
  done
done
echo done
