"""BASELINE.json configurations as plain data (model hyper-parameters + batch
sizes).  Readings C-A3/C-A4/C-A5/C-A22 fix the concrete numbers.

Each entry: ``model`` = keyword overrides of the default npm_config (P:302,
P:305), ``n`` = records per step on one GPU, ``n_global`` = records per
optimisation step over all GPUs of the configuration.
"""

CONFIGS = {
    # configs[0]: 4096 samples, K=8, 4-level 16^3 dense grid, 2x32 MLP
    "c1": dict(model=dict(n_lobes=8, n_levels=4, base_res=2, max_res=16, log2_hashmap=0,
                          mlp_linear_layers=2, mlp_width=32), n=4096, n_global=4096),
    # configs[1]: per-frame batch 1280x720, K=8, multires hash grid, 3x64 MLP
    "c2": dict(model=dict(), n=1280 * 720, n_global=1280 * 720),
    # configs[2]: 8M samples / iteration, 1/2/4/8 GPUs with allreduce
    "c3": dict(model=dict(), n=1 << 23, n_global=1 << 23),
    # configs[3]: product variant, K=16, 4M samples
    "c4": dict(model=dict(mode=1, n_lobes=16), n=1 << 22, n_global=1 << 22),
    # configs[4]: 2^22-entry table x 16 levels, 32M samples / iteration over 8 GPUs
    "c5": dict(model=dict(n_levels=16, base_res=16, max_res=2048, log2_hashmap=22), n=1 << 22,
               n_global=1 << 25),
}

