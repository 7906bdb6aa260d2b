# c4 training-kernel variants, same box: default / ab/<v>.so / env knobs
mkdir -p gpurun_out
T=${TAG:-r02c4ab}
O=gpurun_out/${T}_exp.log
: > $O
run() { echo -n "$1 " >> $O; shift; env "$@" timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {a:round(b['ms']/b['launches']*1000,1) for a,b in d['kernels'].items()})" >> $O; }
for i in 1 2; do
  run wt X=1
  for v in $VARIANTS; do run $v NPM_LIB=$PWD/ab/$v.so; done
  run bintrain NPM_BIN_TRAIN=1
done
echo done
