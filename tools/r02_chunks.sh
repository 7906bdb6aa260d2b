# e2e (npm_frame_step, pinned host buffers) at c2 for NPM_PIPE_CHUNKS = 2 / 3 / 4, same box
mkdir -p gpurun_out
O=gpurun_out/r02chunks_exp.log
: > $O
for i in 1 2; do
  for c in 3 2 4; do
    echo -n "chunks=$c " >> $O
    NPM_PIPE_CHUNKS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value']/1e9,4), round(d['ms_per_step'],4))" >> $O
  done
done
echo done
