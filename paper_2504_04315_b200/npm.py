"""Thin Python binding of the C ABI in include/npm.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of libnpm.so; this module
only converts arrays to pointers.  The functions keep the C names
(npm_create, npm_encode, npm_decode, npm_pdf, npm_sample, npm_train_step, ...);
``Model`` is a small convenience wrapper over them that allocates outputs with
torch (device memory and streams are PyTorch's job, nothing else is).

Arrays may be torch tensors (CUDA or CPU) or numpy arrays: float32,
C-contiguous.  CPU arrays are staged by the library itself (npm.h "POINTERS MAY
BE HOST OR DEVICE").  There is no CPU fallback: if libnpm.so is missing or
fails to load, importing this module raises.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NPM_LIB") or os.path.join(_HERE, "libnpm.so")   # NPM_LIB: A/B builds

RADIANCE, PRODUCT = 0, 1
EXCHANGE_ALLREDUCE, EXCHANGE_ZERO1 = 0, 1
BUF_PARAMS, BUF_GRADS, BUF_ADAM_M, BUF_ADAM_V, BUF_EMA = range(5)
STATUS = {0: "NPM_OK", 1: "NPM_ERR_INVALID", 2: "NPM_ERR_CUDA", 3: "NPM_ERR_NCCL", 4: "NPM_ERR_OOM",
          5: "NPM_ERR_STATE"}


class NpmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class npm_config(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("n_lobes", ctypes.c_int32), ("n_levels", ctypes.c_int32),
                ("n_features", ctypes.c_int32), ("base_res", ctypes.c_int32), ("max_res", ctypes.c_int32),
                ("log2_hashmap", ctypes.c_int32), ("mlp_linear_layers", ctypes.c_int32),
                ("mlp_width", ctypes.c_int32), ("sh_bands", ctypes.c_int32),
                ("aabb_lo", ctypes.c_float * 3), ("aabb_hi", ctypes.c_float * 3),
                ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("adam_eps", ctypes.c_float), ("ema_decay", ctypes.c_float),
                ("kappa_min", ctypes.c_float), ("kappa_max", ctypes.c_float),
                ("init_seed", ctypes.c_uint64), ("divergence", ctypes.c_int32), ("learn_alpha", ctypes.c_int32)]


_FP = ctypes.POINTER(ctypes.c_float)


class npm_query(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64)] + [(k, ctypes.c_void_p) for k in
                                          ("px", "py", "pz", "wox", "woy", "woz", "nx", "ny", "nz", "rough",
                                           "bsdf_pdf")]


class npm_step_stats(ctypes.Structure):
    _fields_ = [("loss_proxy", ctypes.c_double), ("grad_norm_sq", ctypes.c_double),
                ("n_used", ctypes.c_int64), ("n_zero_target", ctypes.c_int64),
                ("n_dropped", ctypes.c_int64), ("n_nonfinite_grad", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libnpm.so not built (run __graft_entry__.build() or "
                          "python paper_2504_04315_b200/build.py): %s" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    V, I64, I32, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64
    M = ctypes.c_void_p
    sig = {
        "npm_default_config": (None, [ctypes.POINTER(npm_config)]),
        "npm_create": (I32, [ctypes.POINTER(npm_config), I32, ctypes.POINTER(M)]),
        "npm_destroy": (I32, [M]),
        "npm_param_count": (I32, [M, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "npm_level_info": (I32, [M, V, V]),
        "npm_get_buffer": (I32, [M, I32, V, I64, V]),
        "npm_set_buffer": (I32, [M, I32, V, I64, V]),
        "npm_get_step": (I32, [M, ctypes.POINTER(I64)]),
        "npm_set_step": (I32, [M, I64]),
        "npm_encode": (I32, [M, ctypes.POINTER(npm_query), I32, V, V]),
        "npm_encode_debug": (I32, [M, ctypes.POINTER(npm_query), V, V, V]),
        "npm_decode": (I32, [M, ctypes.POINTER(npm_query), V, I32, V, V, V, V, V]),
        "npm_pdf": (I32, [M, ctypes.POINTER(npm_query), V, V, V, I32, V, V]),
        "npm_sample": (I32, [M, ctypes.POINTER(npm_query), V, U64, U64, I32, V, V, V, V, V, V, V, V, V]),
        "npm_sample_cosine_product": (I32, [M, ctypes.POINTER(npm_query), V, V, V, ctypes.c_float, V, U64, U64,
                                            I32, V, V, V, V, V, V, V, V, V, V, V, V]),
        "npm_combined_sample": (I32, [M, ctypes.POINTER(npm_query), V, V, V, ctypes.c_float, V, U64, U64, I32,
                                      V, V, V, V, V, V, V]),
        "npm_unwind_records": (I32, [M, V, V, V, V, V, I32, I32, I64, I32, V, V]),
        "npm_train_step": (I32, [M, ctypes.POINTER(npm_query), V, V, V, V, I32, V, I64,
                                 ctypes.POINTER(npm_step_stats), V]),
        "npm_accumulate_grads": (I32, [M, ctypes.POINTER(npm_query), V, V, V, V, I32, V, I64,
                                       ctypes.POINTER(npm_step_stats), V]),
        "npm_train_stream": (I32, [M, ctypes.POINTER(npm_query), V, V, V, V, I32, V, I64,
                                   ctypes.POINTER(npm_step_stats), V]),
        "npm_optimizer_step": (I32, [M, ctypes.POINTER(npm_step_stats), V]),
        "npm_step_stats_async": (I32, [M, ctypes.POINTER(npm_step_stats), V]),
        "npm_frame_step": (I32, [M, ctypes.POINTER(npm_query), V, U64, U64, I32, V, V, V, V, V, V, V, V,
                                 ctypes.POINTER(npm_query), V, V, V, V, I32, V, I64, ctypes.POINTER(npm_step_stats), V]),
        "npm_get_unique_id": (I32, [V]),
        "npm_set_exchange": (I32, [M, I32]),
        "npm_shard_range": (I32, [M, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "npm_optimizer_step_shard": (I32, [M, I32, I32, ctypes.POINTER(npm_step_stats), V]),
        "npm_ema_update": (I32, [M, V]),
        "npm_comm_init": (I32, [M, I32, I32, V]),
        "npm_buffer_device_ptr": (I32, [M, I32, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(I64)]),
        "npm_launch_count": (I64, [M]),
        "npm_profile_kinds": (I32, []),
        "npm_profile_enable": (I32, [M, I32]),
        "npm_profile_reset": (I32, [M]),
        "npm_profile_read": (I32, [M, I32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(I64),
                                   ctypes.POINTER(ctypes.c_double)]),
        "npm_probe_grid_access": (I32, [I32, I64, I64, I32, I32, I32, ctypes.POINTER(ctypes.c_double)]),
        "npm_abi_sizes": (None, [ctypes.POINTER(I32)] * 3),
        "npm_last_error": (ctypes.c_char_p, []),
        "npm_version": (I32, []),
    }
    optional = {"npm_probe_grid_access", "npm_abi_sizes", "npm_step_stats_async", "npm_get_unique_id",
                "npm_comm_init"}   # absent in older A/B builds
    for name, (res, args) in sig.items():
        if name in optional and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_lib = _load()


def npm_abi_sizes():
    c, q, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.npm_abi_sizes(ctypes.byref(c), ctypes.byref(q), ctypes.byref(s))
    return c.value, q.value, s.value


if hasattr(_lib, "npm_abi_sizes") and npm_abi_sizes() != (ctypes.sizeof(npm_config), ctypes.sizeof(npm_query),
                                                           ctypes.sizeof(npm_step_stats)):
    raise ImportError("libnpm.so struct layout does not match this binding (rebuild the library)")

# ---------------------------------------------------------------------------
# raw C-name wrappers


def _check(st):
    if st != 0:
        raise NpmError(st, _lib.npm_last_error().decode())


def _ptr(x):
    """Pointer of a float32/uint32 C-contiguous torch tensor or numpy array."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    if not x.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        return None
    return ctypes.c_void_p(stream)


def npm_default_config(**overrides):
    c = npm_config()
    _lib.npm_default_config(ctypes.byref(c))
    for k, v in overrides.items():
        if k in ("aabb_lo", "aabb_hi"):
            setattr(c, k, (ctypes.c_float * 3)(*v))
        else:
            setattr(c, k, v)
    return c


def npm_create(cfg, device=0):
    h = ctypes.c_void_p()
    _check(_lib.npm_create(ctypes.byref(cfg), int(device), ctypes.byref(h)))
    return h


def npm_destroy(h):
    _check(_lib.npm_destroy(h))


def make_query(n, px, py, pz, wox=None, woy=None, woz=None, nx=None, ny=None, nz=None, rough=None, bsdf_pdf=None):
    q = npm_query()
    q.n = int(n)
    for k, v in zip(("px", "py", "pz", "wox", "woy", "woz", "nx", "ny", "nz", "rough", "bsdf_pdf"),
                    (px, py, pz, wox, woy, woz, nx, ny, nz, rough, bsdf_pdf)):
        setattr(q, k, _ptr(v))
    return q


def npm_encode(h, q, use_ema, feat, stream=None):
    _check(_lib.npm_encode(h, ctypes.byref(q), int(use_ema), _ptr(feat), _stream(stream)))


def npm_encode_debug(h, q, idx, w, stream=None):
    _check(_lib.npm_encode_debug(h, ctypes.byref(q), _ptr(idx), _ptr(w), _stream(stream)))


def npm_decode(h, q, feat, use_ema, raw, lam, kappa, mu, stream=None):
    _check(_lib.npm_decode(h, ctypes.byref(q), _ptr(feat), int(use_ema), _ptr(raw), _ptr(lam), _ptr(kappa),
                           _ptr(mu), _stream(stream)))


def npm_pdf(h, q, wx, wy, wz, use_ema, pdf, stream=None):
    _check(_lib.npm_pdf(h, ctypes.byref(q), _ptr(wx), _ptr(wy), _ptr(wz), int(use_ema), _ptr(pdf),
                        _stream(stream)))


def npm_sample(h, q, u, seed, offset, use_ema, wx, wy, wz, pdf, qx=None, qy=None, qz=None, pdf_q=None,
               stream=None):
    _check(_lib.npm_sample(h, ctypes.byref(q), _ptr(u), int(seed), int(offset), int(use_ema), _ptr(wx),
                           _ptr(wy), _ptr(wz), _ptr(pdf), _ptr(qx), _ptr(qy), _ptr(qz), _ptr(pdf_q),
                           _stream(stream)))


def npm_train_stream(h, q, wx, wy, wz, target, channels, spdf, micro_batch, want_stats=True, stream=None):
    steps = (q.n + micro_batch - 1) // micro_batch if micro_batch > 0 else 0
    arr = (npm_step_stats * max(steps, 1))() if want_stats else None
    _check(_lib.npm_train_stream(h, ctypes.byref(q), _ptr(wx), _ptr(wy), _ptr(wz), _ptr(target), int(channels),
                                 _ptr(spdf), int(micro_batch), arr, _stream(stream)))
    return [arr[i].as_dict() for i in range(steps)] if want_stats else None


def npm_sample_cosine_product(h, q, nx, ny, nz, kappa_c, u, seed, offset, use_ema, wx, wy, wz, pdf, qx=None, qy=None,
                              qz=None, pdf_q=None, lam=None, kappa=None, mu=None, stream=None):
    _check(_lib.npm_sample_cosine_product(h, ctypes.byref(q), _ptr(nx), _ptr(ny), _ptr(nz), float(kappa_c), _ptr(u),
                                          int(seed), int(offset), int(use_ema), _ptr(wx), _ptr(wy), _ptr(wz), _ptr(pdf),
                                          _ptr(qx), _ptr(qy), _ptr(qz), _ptr(pdf_q), _ptr(lam), _ptr(kappa), _ptr(mu),
                                          _stream(stream)))


def npm_get_unique_id():
    """128-byte NCCL unique id (rank 0 creates it, every rank passes it to npm_comm_init)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.npm_get_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def npm_comm_init(h, rank, world, uid):
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(_lib.npm_comm_init(h, int(rank), int(world), ctypes.cast(buf, ctypes.c_void_p)))


def npm_step_stats_async(h, out_ptr, stream=None):
    """out_ptr: address of an npm_step_stats in pinned host memory (e.g. a
    pinned torch uint8 tensor of ctypes.sizeof(npm_step_stats) bytes)."""
    _check(_lib.npm_step_stats_async(h, ctypes.cast(out_ptr, ctypes.POINTER(npm_step_stats)), _stream(stream)))


def npm_combined_sample(h, q, nx, ny, nz, alpha, u, seed, offset, use_ema, wx, wy, wz, pdf, guide_pdf=None,
                        technique=None, stream=None):
    _check(_lib.npm_combined_sample(h, ctypes.byref(q), _ptr(nx), _ptr(ny), _ptr(nz), float(alpha), _ptr(u),
                                    int(seed), int(offset), int(use_ema), _ptr(wx), _ptr(wy), _ptr(wz), _ptr(pdf),
                                    _ptr(guide_pdf), _ptr(technique), _stream(stream)))


def npm_unwind_records(h, le, fs, cos_theta, pdf, depth, channels, max_depth, n_paths, product, target,
                       stream=None):
    _check(_lib.npm_unwind_records(h, _ptr(le), _ptr(fs), _ptr(cos_theta), _ptr(pdf), _ptr(depth), int(channels),
                                   int(max_depth), int(n_paths), int(product), _ptr(target), _stream(stream)))


def npm_train_step(h, q, wx, wy, wz, target, channels, spdf, n_global, want_stats=True, stream=None):
    st = npm_step_stats() if want_stats else None
    _check(_lib.npm_train_step(h, ctypes.byref(q), _ptr(wx), _ptr(wy), _ptr(wz), _ptr(target), int(channels),
                               _ptr(spdf), int(n_global), ctypes.byref(st) if st is not None else None,
                               _stream(stream)))
    return st.as_dict() if st is not None else None


def npm_accumulate_grads(h, q, wx, wy, wz, target, channels, spdf, n_global, want_stats=True, stream=None):
    st = npm_step_stats() if want_stats else None
    _check(_lib.npm_accumulate_grads(h, ctypes.byref(q), _ptr(wx), _ptr(wy), _ptr(wz), _ptr(target),
                                     int(channels), _ptr(spdf), int(n_global),
                                     ctypes.byref(st) if st is not None else None, _stream(stream)))
    return st.as_dict() if st is not None else None


def npm_optimizer_step(h, want_stats=True, stream=None):
    st = npm_step_stats() if want_stats else None
    _check(_lib.npm_optimizer_step(h, ctypes.byref(st) if st is not None else None, _stream(stream)))
    return st.as_dict() if st is not None else None


def npm_frame_step(h, q, u, seed, offset, use_ema, wx, wy, wz, pdf, qx, qy, qz, pdf_q, tq, twx, twy, twz, target,
                   channels, spdf, n_global, want_stats=True, stream=None):
    st = npm_step_stats() if want_stats else None
    _check(_lib.npm_frame_step(h, ctypes.byref(q), _ptr(u), int(seed), int(offset), int(use_ema), _ptr(wx), _ptr(wy),
                               _ptr(wz), _ptr(pdf), _ptr(qx), _ptr(qy), _ptr(qz), _ptr(pdf_q), ctypes.byref(tq),
                               _ptr(twx), _ptr(twy), _ptr(twz), _ptr(target), int(channels), _ptr(spdf),
                               int(n_global), ctypes.byref(st) if st is not None else None, _stream(stream)))
    return st.as_dict() if st is not None else None


def npm_set_exchange(h, mode):
    _check(_lib.npm_set_exchange(h, int(mode)))


def npm_shard_range(h, rank, world):
    """(begin, count, chunk) of rank's ZeRO-1 shard of the flat parameter vector."""
    b, c, ch = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.npm_shard_range(h, int(rank), int(world), ctypes.byref(b), ctypes.byref(c), ctypes.byref(ch)))
    return b.value, c.value, ch.value


def npm_optimizer_step_shard(h, rank, world, want_stats=True, stream=None):
    st = npm_step_stats() if want_stats else None
    _check(_lib.npm_optimizer_step_shard(h, int(rank), int(world), ctypes.byref(st) if st is not None else None,
                                         _stream(stream)))
    return st.as_dict() if st is not None else None


def npm_ema_update(h, stream=None):
    _check(_lib.npm_ema_update(h, _stream(stream)))


def npm_param_count(h):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.npm_param_count(h, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def npm_level_info(h, n_levels):
    res = np.zeros(n_levels, np.int32)
    ent = np.zeros(n_levels, np.int64)
    _check(_lib.npm_level_info(h, res.ctypes.data, ent.ctypes.data))
    return res, ent


def npm_get_buffer(h, which, dst, stream=None):
    _check(_lib.npm_get_buffer(h, int(which), _ptr(dst), int(dst.numel() if hasattr(dst, "numel") else dst.size),
                               _stream(stream)))


def npm_set_buffer(h, which, src, stream=None):
    _check(_lib.npm_set_buffer(h, int(which), _ptr(src), int(src.numel() if hasattr(src, "numel") else src.size),
                               _stream(stream)))


def npm_get_step(h):
    t = ctypes.c_int64()
    _check(_lib.npm_get_step(h, ctypes.byref(t)))
    return t.value


def npm_set_step(h, t):
    _check(_lib.npm_set_step(h, int(t)))


def npm_buffer_device_ptr(h, which):
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(_lib.npm_buffer_device_ptr(h, int(which), ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def npm_launch_count(h):
    return int(_lib.npm_launch_count(h))


def npm_profile_enable(h, on):
    _check(_lib.npm_profile_enable(h, int(on)))


def npm_profile_reset(h):
    _check(_lib.npm_profile_reset(h))


def npm_probe_grid_access(device, table_entries, n_samples, levels, kind, reps=5):
    """Mean ms per launch of the random grid-access probe (include/npm.h)."""
    ms = ctypes.c_double()
    _check(_lib.npm_probe_grid_access(device, table_entries, n_samples, levels, kind, reps, ctypes.byref(ms)))
    return ms.value


def npm_profile_read(h):
    """{kernel kind: (launches, total_ms)} since the last reset."""
    out = {}
    for k in range(_lib.npm_profile_kinds()):
        name, n, ms = ctypes.c_char_p(), ctypes.c_int64(), ctypes.c_double()
        _check(_lib.npm_profile_read(h, k, ctypes.byref(name), ctypes.byref(n), ctypes.byref(ms)))
        out[name.value.decode()] = (n.value, ms.value)
    return out


# ---------------------------------------------------------------------------
# Convenience wrapper with torch-allocated outputs.


class _CudaArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


class Model:
    def __init__(self, device=0, **cfg):
        import torch
        self.torch = torch
        self.cfg = npm_default_config(**cfg)
        self.device = torch.device("cuda", device)
        self.h = npm_create(self.cfg, device)
        self.n_grid, self.n_mlp = npm_param_count(self.h)
        self.n_alpha = (self.cfg.mlp_width + 1 + 3) // 4 * 4 if self.cfg.learn_alpha else 0
        self.n_params = self.n_grid + self.n_mlp + self.n_alpha
        self.K = self.cfg.n_lobes
        self.L = self.cfg.n_levels
        self.F = self.cfg.n_features
        self.product = self.cfg.mode == PRODUCT

    def close(self):
        if self.h:
            npm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _f32(self, x):
        t = self.torch
        if x is None:
            return None
        if isinstance(x, np.ndarray):
            x = t.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        return x.to(device=self.device, dtype=t.float32).contiguous()

    def _empty(self, *shape, dtype=None):
        return self.torch.empty(*shape, device=self.device, dtype=dtype or self.torch.float32)

    def query(self, x, wo=None, nrm=None, rough=None, bsdf_pdf=None):
        """x: [3, n]; product mode also wo [3, n], nrm [3, n], rough [n];
        bsdf_pdf [n]: training records of a learn_alpha model (C-A34)."""
        x = self._f32(x)
        pb = self._f32(bsdf_pdf)
        keep = [x, pb]
        if self.product:
            wo, nrm, rough = self._f32(wo), self._f32(nrm), self._f32(rough)
            keep += [wo, nrm, rough]
            q = make_query(x.shape[1], x[0], x[1], x[2], wo[0], wo[1], wo[2], nrm[0], nrm[1], nrm[2], rough, pb)
        else:
            q = make_query(x.shape[1], x[0], x[1], x[2], bsdf_pdf=pb)
        q._keep = keep
        return q

    def buffer_view(self, which, count=None):
        """Zero-copy torch view of a model buffer (e.g. GRADS for a collective);
        count > n_params views the zero padding too (<= n_params + 264, the
        ZeRO-1 world * chunk of npm_shard_range)."""
        p, n = npm_buffer_device_ptr(self.h, which)
        if count is not None:
            if count > n + 264:
                raise ValueError("view beyond the buffer's padding")
            n = count
        return self.torch.as_tensor(_CudaArray(p, n), device=self.device)

    def get(self, which=BUF_PARAMS):
        out = self._empty(self.n_params)
        npm_get_buffer(self.h, which, out, self._stream())
        return out

    def set(self, which, values):
        v = self._f32(values)
        npm_set_buffer(self.h, which, v, self._stream())

    def encode(self, q, use_ema=False):
        feat = self._empty(self.L * self.F, q.n)
        npm_encode(self.h, q, use_ema, feat, self._stream())
        return feat

    def encode_debug(self, q):
        idx = self._empty(self.L, 8, q.n, dtype=self.torch.int32)
        w = self._empty(self.L, 8, q.n)
        npm_encode_debug(self.h, q, idx, w, self._stream())
        return idx, w

    def decode(self, q, use_ema=False, feat=None):
        n = q.n
        raw, lam, kap, mu = (self._empty(4 * self.K, n), self._empty(self.K, n), self._empty(self.K, n),
                             self._empty(3, self.K, n))
        npm_decode(self.h, q, self._f32(feat), use_ema, raw, lam, kap, mu, self._stream())
        return raw, lam, kap, mu

    def pdf(self, q, w, use_ema=False):
        w = self._f32(w)
        out = self._empty(q.n)
        npm_pdf(self.h, q, w[0], w[1], w[2], use_ema, out, self._stream())
        return out

    def sample(self, q, u=None, seed=0, offset=0, use_ema=False, wq=None):
        n = q.n
        wi, pdf = self._empty(3, n), self._empty(n)
        u = self._f32(u)
        if wq is not None:
            wq = self._f32(wq)
            pdf_q = self._empty(n)
            npm_sample(self.h, q, u, seed, offset, use_ema, wi[0], wi[1], wi[2], pdf, wq[0], wq[1], wq[2], pdf_q,
                       stream=self._stream())
            return wi, pdf, pdf_q
        npm_sample(self.h, q, u, seed, offset, use_ema, wi[0], wi[1], wi[2], pdf, stream=self._stream())
        return wi, pdf

    def combined_sample(self, q, nrm, alpha=0.5, u=None, seed=0, offset=0, use_ema=False):
        """f-1 one-sample MIS of the BSDF stand-in and the guide.  nrm: unit
        shading normals [3, n]; u: [4, n] or None (Philox).  Returns
        (wi [3, n], p~ [n], V(wi) [n], technique int32 [n])."""
        n = q.n
        nrm, u = self._f32(nrm), self._f32(u)
        wi, pdf, gpdf = self._empty(3, n), self._empty(n), self._empty(n)
        tech = self._empty(n, dtype=self.torch.int32)
        npm_combined_sample(self.h, q, nrm[0], nrm[1], nrm[2], alpha, u, seed, offset, use_ema, wi[0], wi[1], wi[2],
                            pdf, gpdf, tech, stream=self._stream())
        return wi, pdf, gpdf, tech

    def sample_cosine_product(self, q, nrm, kappa_c=2.1438, u=None, seed=0, offset=0, use_ema=False, wq=None):
        """f-2: sample / pdf of the mixture times the cosine lobe about nrm.
        Returns (wi [3, n], pdf [n], pdf_q [n] or None, lambda [K, n],
        kappa [K, n], mu [3, K, n]) of the product mixture."""
        n, K = q.n, self.K
        nrm, u = self._f32(nrm), self._f32(u)
        wi, pdf = self._empty(3, n), self._empty(n)
        lam, kap, mu = self._empty(K, n), self._empty(K, n), self._empty(3, K, n)
        pdf_q = None
        qx = qy = qz = None
        if wq is not None:
            wq = self._f32(wq)
            qx, qy, qz = wq[0], wq[1], wq[2]
            pdf_q = self._empty(n)
        npm_sample_cosine_product(self.h, q, nrm[0], nrm[1], nrm[2], kappa_c, u, seed, offset, use_ema, wi[0], wi[1],
                                  wi[2], pdf, qx, qy, qz, pdf_q, lam, kap, mu, stream=self._stream())
        return wi, pdf, pdf_q, lam, kap, mu

    def unwind_records(self, le, fs, cos_theta, pdf, depth, product=False):
        """f-1 training-record unwind: le, fs [C, D, n]; cos_theta, pdf [D, n];
        depth int32 [n] -> D^ [C, D, n]."""
        le, fs, cos_theta, pdf = self._f32(le), self._f32(fs), self._f32(cos_theta), self._f32(pdf)
        t = self.torch
        depth = (t.from_numpy(np.ascontiguousarray(depth, dtype=np.int32)) if isinstance(depth, np.ndarray)
                 else depth).to(device=self.device, dtype=t.int32).contiguous()
        C, D, n = le.shape
        out = self._empty(C, D, n)
        npm_unwind_records(self.h, le, fs, cos_theta, pdf, depth, C, D, n, int(product), out, stream=self._stream())
        return out

    def train_stream(self, q, wi, target, spdf, micro_batch=1 << 18, want_stats=True):
        """f-3: one optimisation step per consecutive micro-batch of the records."""
        wi, target, spdf = self._train_args(wi, target, spdf)
        return npm_train_stream(self.h, q, wi[0], wi[1], wi[2], target, target.shape[0], spdf, micro_batch,
                                want_stats, self._stream())

    def _train_args(self, wi, target, spdf):
        wi, target, spdf = self._f32(wi), self._f32(target), self._f32(spdf)
        if target.dim() == 1:
            target = target[None]
        return wi, target, spdf

    def train_step(self, q, wi, target, spdf, n_global=None, want_stats=True):
        wi, target, spdf = self._train_args(wi, target, spdf)
        return npm_train_step(self.h, q, wi[0], wi[1], wi[2], target, target.shape[0], spdf,
                              q.n if n_global is None else n_global, want_stats, self._stream())

    def accumulate_grads(self, q, wi, target, spdf, n_global=None, want_stats=True):
        wi, target, spdf = self._train_args(wi, target, spdf)
        return npm_accumulate_grads(self.h, q, wi[0], wi[1], wi[2], target, target.shape[0], spdf,
                                    q.n if n_global is None else n_global, want_stats, self._stream())

    def optimizer_step(self, want_stats=True):
        return npm_optimizer_step(self.h, want_stats, self._stream())

    @property
    def step(self):
        return npm_get_step(self.h)

    @step.setter
    def step(self, t):
        npm_set_step(self.h, t)

    @property
    def launches(self):
        return npm_launch_count(self.h)

    def level_info(self):
        return npm_level_info(self.h, self.L)
