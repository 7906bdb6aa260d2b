# round-2 full GPU check + phase stamps
set -x
mkdir -p gpurun_out
T=${TAG:-r02p}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
for v in shuffled sorted; do NPM_DEBUG=4 timeout 120 python tools/train_exp.py $v 2>&1 | grep -E "NPM_|variant" | tail -3 >> gpurun_out/${T}_phase.log; done
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo done
