# bench lines for every configuration (one GPU); outputs under gpurun_out/
python bench.py --steps 20 --warmup 5 > gpurun_out/all_c2.json 2> gpurun_out/all_c2.err
for w in c1 c3 c4 c5; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/all_$w.json 2>/dev/null; done
python - <<'PY'
import json
for w in ["c1","c2","c3","c4","c5"]:
    try:
        d=json.loads(open("gpurun_out/all_%s.json"%w).read().strip().splitlines()[-1])
    except Exception as e:
        print(w, "ERR", e); continue
    r=d["roofline"]
    print(w, "%.4f ms"%d["ms_per_step"], "val %.3g train %.3g q %.3g e2e %.3g"%(d["value"],d["train_samples_per_s"],d["queries_per_s"],d["e2e"]["value"]),
          "frac %.3f"%r["frac"], {k:round(v["ms"]/v["launches"]*1000,1) for k,v in d["kernels"].items()}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"],
          "cpu", (d.get("cpu_baseline") or {}).get("value"), "probe", {k:round(v,3) for k,v in r.get("grid_access_probe",{}).items() if "frac" in k})
PY
