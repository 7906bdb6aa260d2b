ab() { # variants...
for i in 1 2; do for v in "$@"; do NPM_LIB=$PWD/ab/libnpm_$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v\", round(d[\"ms_per_step\"],4), {a:round(b[\"ms\"]/b[\"launches\"]*1000,1) for a,b in d[\"kernels\"].items()})"; done; done
}
# per-phase clock stamps (CTA 0, group 0) of one training launch: ab_phases variant
ab_phases() {
for v in "$@"; do echo -n "$v "; NPM_LIB=$PWD/ab/libnpm_$v.so NPM_DEBUG=4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep NPM_PHASES | tail -1; done
}
# c5 / p16 workloads
ab_w() { # workload variants...
w=$1; shift
for i in 1 2; do for v in "$@"; do NPM_LIB=$PWD/ab/libnpm_$v.so python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$w $v\", round(d[\"ms_per_step\"],4), {a:round(b[\"ms\"]/b[\"launches\"]*1000,1) for a,b in d[\"kernels\"].items()})"; done; done
}
