# round-2 GPU check: full gpu test suite + smoke + default bench
set -x
mkdir -p gpurun_out
T=${TAG:-r02a}
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo done
