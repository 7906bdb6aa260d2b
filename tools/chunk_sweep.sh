mkdir -p gpurun_out
timeout 120 python tools/link_probe.py > gpurun_out/link_probe.json 2> gpurun_out/link_probe.err
for r in 1 2; do for c in 3 4; do NPM_PIPE_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/sweep3_c${c}_$r.json 2>/dev/null; done; done
echo done
