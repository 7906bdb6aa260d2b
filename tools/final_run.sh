set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01f_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/r01f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r01f_smoke.log
timeout 600 python bench.py > gpurun_out/r01f_bench_default.json 2> gpurun_out/r01f_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01f_bench_reference.json 2> gpurun_out/r01f_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r01f_ncu_launch.log 2>&1
echo done
