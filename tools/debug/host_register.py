import ctypes, time, numpy as np, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
import glob, os
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
a = np.random.rand(4, 987, 3072)  # 97 MB
d = torch.empty(a.size, dtype=torch.float64, device="cuda")
for trial in range(3):
    t0 = time.perf_counter()
    r = rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 0)
    t1 = time.perf_counter()
    rt.cudaMemcpy(ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(a.nbytes), 1)
    t2 = time.perf_counter()
    rt.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
    t3 = time.perf_counter()
    print("rc", r, "register %.2f ms copy %.2f ms unregister %.2f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3))
