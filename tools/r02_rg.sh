# radiance query in one chain group (ab/rg1.so) vs two (working tree), same box
mkdir -p gpurun_out
T=${TAG:-r02rg}
O=gpurun_out/${T}_exp.log
: > $O
for i in 1 2; do
  for v in wt rg1; do
    L=X=1; [ $v != wt ] && L=NPM_LIB=$PWD/ab/$v.so
    for w in c2 c5; do echo -n "$v $w " >> $O; env $L EXP_WORKLOAD=$w timeout 150 python tools/query_exp.py 2>&1 | tail -1 >> $O; done
    echo -n "$v f1f2 " >> $O; env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-strong 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['f1_guided_mis']['combined_sample_ms'], d['f2_cosine_product']['cosine_product_sample_plus_pdf_ms'])" >> $O
  done
done
echo done
