# c5 training: the r01 kernel (default) vs the warp-specialised kernel
# (NPM_TRAIN_WS=1, binned + privatised scatter) with gather variants ab/<v>.so
mkdir -p gpurun_out
T=${TAG:-r02c5ab}
O=gpurun_out/${T}_exp.log
: > $O
run() { echo -n "$1 " >> $O; shift; env "$@" timeout 300 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O; }
for i in 1 2; do
  run r01 X=1
  run ws NPM_TRAIN_WS=1
  for v in $VARIANTS; do run $v NPM_TRAIN_WS=1 NPM_LIB=$PWD/ab/$v.so; done
done
echo done
