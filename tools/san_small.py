import numpy as np, sys
sys.path.insert(0, '.')
from paper_2504_04315_b200 import npm
from workloads import synth
from workloads.configs import CONFIGS
for name in ("c2", "c4"):
    m = npm.Model(0, **CONFIGS[name]["model"])
    prod = m.product
    b = synth.training_batch(70000, seed=1, product=prod)
    q = m.query(b["x"], b["wo"], b["nrm"], b["rough"])
    m.train_step(q, b["wi"], b["target"], b["pdf"])
    qb = synth.query_batch(70000, seed=2, product=prod)
    qq = m.query(qb["x"], qb["wo"], qb["nrm"], qb["rough"])
    m.sample(qq, seed=1, wq=qb["wq"])
    m.decode(qq); m.pdf(qq, qb["wq"]); m.encode(qq)
    print(name, "ok")
