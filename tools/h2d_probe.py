"""Host <-> device copy bandwidth of this box, the ceiling of bench.py's e2e
number: pinned host buffers, cudaMemcpyAsync on each GPU's own copy streams,
GPUs alone and all together, H2D alone and H2D + D2H together (what one
e2e step does: 2 operands in, 1 result out).  Wall clock around device-synced
copies; prints GB/s."""
import sys
import threading
import time

import torch

GB = 1e9
n_gpu = torch.cuda.device_count()
size = int(float(sys.argv[1]) * 2**30) if len(sys.argv) > 1 else 2**31  # bytes per buffer
bufs = []
for d in range(n_gpu):
    h_in = torch.empty(size // 4, dtype=torch.float32).pin_memory()
    h_out = torch.empty(size // 4, dtype=torch.float32).pin_memory()
    dev_in = torch.empty(size // 4, dtype=torch.float32, device=f"cuda:{d}")
    dev_out = torch.empty(size // 4, dtype=torch.float32, device=f"cuda:{d}")
    s_in = torch.cuda.Stream(device=d)
    s_out = torch.cuda.Stream(device=d)
    bufs.append((h_in, h_out, dev_in, dev_out, s_in, s_out))


def run(gpus, h2d=True, d2h=False, reps=3):
    def one(d):
        h_in, h_out, dev_in, dev_out, s_in, s_out = bufs[d]
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s_in):
                    dev_in.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s_out):
                    h_out.copy_(dev_out, non_blocking=True)
        s_in.synchronize()
        s_out.synchronize()
    for d in gpus:  # warm
        one(d)
    t0 = time.perf_counter()
    th = [threading.Thread(target=one, args=(d,)) for d in gpus]
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    moved = size * reps * len(gpus) * ((1 if h2d else 0) + (1 if d2h else 0))
    return moved / dt / GB


def run2d(gpus, h2d=True, d2h=False, reps=3):
    """The same bytes as row-pitched 2-D copies: rows of size/2 bytes... here
    16384-float rows out of 32768-float host rows (a checkerboard block of a
    row-major host matrix, as scatter / gather copy it)."""
    import ctypes
    import glob
    import os
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    libs += glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                   "libcudart.so*"))
    rt = ctypes.CDLL(libs[0])
    width = 16384 * 4
    height = size // width
    host_pitch = 2 * width
    hosts = [torch.empty(height * host_pitch // 4, dtype=torch.float32).pin_memory() for _ in gpus]

    def one(i, d):
        h_in, h_out, dev_in, dev_out, s_in, s_out = bufs[d]
        torch.cuda.set_device(d)
        for _ in range(reps):
            if h2d:
                rt.cudaMemcpy2DAsync(ctypes.c_void_p(dev_in.data_ptr()), ctypes.c_size_t(width),
                                     ctypes.c_void_p(hosts[i].data_ptr()), ctypes.c_size_t(host_pitch),
                                     ctypes.c_size_t(width), ctypes.c_size_t(height), 1,
                                     ctypes.c_void_p(s_in.cuda_stream))
            if d2h:
                rt.cudaMemcpy2DAsync(ctypes.c_void_p(hosts[i].data_ptr()), ctypes.c_size_t(host_pitch),
                                     ctypes.c_void_p(dev_out.data_ptr()), ctypes.c_size_t(width),
                                     ctypes.c_size_t(width), ctypes.c_size_t(height), 2,
                                     ctypes.c_void_p(s_out.cuda_stream))
        s_in.synchronize()
        s_out.synchronize()
    for i, d in enumerate(gpus):
        one(i, d)
    t0 = time.perf_counter()
    th = [threading.Thread(target=one, args=(i, d)) for i, d in enumerate(gpus)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.perf_counter() - t0
    moved = width * height * reps * len(gpus) * ((1 if h2d else 0) + (1 if d2h else 0))
    return moved / dt / GB


print(f"{n_gpu} GPUs, {size / 2**30:.1f} GiB buffers")
for gpus in ([0], list(range(n_gpu))):
    for h2d, d2h in ((True, False), (False, True), (True, True)):
        tag = ("H2D" if h2d else "") + ("+" if h2d and d2h else "") + ("D2H" if d2h else "")
        print(f"gpus={len(gpus)} {tag:8s} {run(gpus, h2d, d2h):7.1f} GB/s aggregate", flush=True)
for gpus in ([0], list(range(n_gpu))):
    for h2d, d2h in ((True, False), (False, True), (True, True)):
        tag = ("H2D" if h2d else "") + ("+" if h2d and d2h else "") + ("D2H" if d2h else "")
        print(f"gpus={len(gpus)} {tag:8s} {run2d(gpus, h2d, d2h):7.1f} GB/s aggregate (2-D, 64 KB rows, 128 KB host pitch)",
              flush=True)
