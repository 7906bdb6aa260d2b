# HEAD verification: GPU tests, smoke, bench lines for c2 / c4 / c5
mkdir -p gpurun_out
T=${TAG:-r02x}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
for w in c4 c5; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-strong > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; done
echo done
