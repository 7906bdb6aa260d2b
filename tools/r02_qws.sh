# query_ws check: parity suites on the sample / pdf path, then same-box timing
# with the warp-specialised kernel on / off
mkdir -p gpurun_out
T=${TAG:-r02qws}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kappa_edges.py tests/test_gpu_guide.py tests/test_gpu_pipeline.py -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for w in 1 0; do echo -n "qws=$w " >> $O; NPM_QUERY_WS=$w timeout 300 python tools/query_exp.py 2>&1 | tail -1 >> $O; done
  echo -n "c5 qws=1 " >> $O; EXP_WORKLOAD=c5 NPM_QUERY_WS=1 timeout 300 python tools/query_exp.py 2>&1 | tail -1 >> $O
  echo -n "c5 qws=0 " >> $O; EXP_WORKLOAD=c5 NPM_QUERY_WS=0 timeout 300 python tools/query_exp.py 2>&1 | tail -1 >> $O
done
echo done
