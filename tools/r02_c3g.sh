# c3 (2^23 queries, L2-resident tables): two chain groups (default) vs one (NPM_QWS_GROUPS=1)
mkdir -p gpurun_out
O=gpurun_out/r02c3g_exp.log
: > $O
for i in 1 2; do
  for g in 2 1; do
    echo -n "groups=$g " >> $O
    NPM_QWS_GROUPS=$g timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O
  done
done
echo done
