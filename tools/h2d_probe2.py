"""H2D bandwidth of the e2e input size: pinned (cached) vs write-combined host
memory, one vs two copy streams (cudart via ctypes)."""
import ctypes, glob, os
import torch
torch.cuda.init()
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
n = 16_411_928
d = torch.empty(n // 8, dtype=torch.int64, device="cuda")
def host(flags):
    p = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), ctypes.c_uint(flags)) == 0
    ctypes.memset(p, 1, n)
    return p
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=30):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for name, flags in (("cached pinned", 0), ("write-combined", 4), ("portable", 1)):
    p = host(flags)
    one = lambda: rt.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr()), p, ctypes.c_size_t(n), 1,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    def two():
        cur = torch.cuda.current_stream(); s1.wait_stream(cur); s2.wait_stream(cur)
        h = n // 2
        rt.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr()), p, ctypes.c_size_t(h), 1, ctypes.c_void_p(s1.cuda_stream))
        rt.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr() + h), ctypes.c_void_p(p.value + h), ctypes.c_size_t(n - h), 1,
                           ctypes.c_void_p(s2.cuda_stream))
        cur.wait_stream(s1); cur.wait_stream(s2)
    t1, t2 = timeit(one), timeit(two)
    print(f"{name:15s} 1 stream {t1*1e3:7.1f} us ({n/t1/1e6:5.1f} GB/s)  2 streams {t2*1e3:7.1f} us ({n/t2/1e6:5.1f} GB/s)")
