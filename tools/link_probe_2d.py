"""Host link probe, pipeline-shaped: the c2 e2e step's copies issued exactly
as HostPipe does (3 chunks, one cudaMemcpy2DAsync per host array per chunk,
H2D on one stream, D2H on another), no kernels.  Prints one JSON line."""
import ctypes, glob, json, os
import torch

lib = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(lib[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]

n, chunks = 921600, int(os.environ.get("CHUNKS", "3"))
C = (n + chunks - 1) // chunks
dev = torch.device("cuda:0")
h2d_arrays = [3, 3] + [3, 3, 1, 1]          # query x, wq; train x, wi, target (1 channel), pdf
# (profiles/r01f_link_probe_2d.json was taken with a 3-channel target: 16 floats/sample of H2D)
d2h_arrays = [3, 1, 1]                       # wi, pdf, pdf_q
hin = [torch.empty(c * n, dtype=torch.float32).pin_memory() for c in h2d_arrays]
din = [torch.empty(c * n, dtype=torch.float32, device=dev) for c in h2d_arrays]
hout = [torch.empty(c * n, dtype=torch.float32).pin_memory() for c in d2h_arrays]
dout = [torch.empty(c * n, dtype=torch.float32, device=dev) for c in d2h_arrays]
cs, ds = torch.cuda.Stream(), torch.cuda.Stream()

def step(with_d2h=True):
    for j in range(chunks):
        c = min(C, n - j * C)
        for k, comps in enumerate(h2d_arrays):
            assert rt.cudaMemcpy2DAsync(din[k].data_ptr() + j * C * comps * 4, c * 4, hin[k].data_ptr() + j * C * 4,
                                        n * 4, c * 4, comps, 1, cs.cuda_stream) == 0
        if with_d2h:
            for k, comps in enumerate(d2h_arrays):
                assert rt.cudaMemcpy2DAsync(hout[k].data_ptr() + j * C * 4, n * 4, dout[k].data_ptr() + j * C * comps * 4,
                                            c * 4, c * 4, comps, 2, ds.cuda_stream) == 0

def timed(with_d2h, reps=20):
    for _ in range(3):
        step(with_d2h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    ds.wait_stream(cs)
    for _ in range(reps):
        step(with_d2h)
    cs.wait_stream(ds)
    e1.record(cs)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

print(json.dumps({"chunks": chunks, "h2d_2d_ms_per_step": timed(False), "h2d_plus_d2h_2d_ms_per_step": timed(True),
                  "h2d_bytes": 4 * n * sum(h2d_arrays), "d2h_bytes": 4 * n * sum(d2h_arrays)}))
