import ctypes, time, glob, torch
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
libs = glob.glob('/usr/local/cuda/lib64/libcudart.so*') + glob.glob('/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*')
rt = ctypes.CDLL(libs[0])
res = []
for rep in range(3):
    for mb in (256, 1024, 4096):
        p = ctypes.c_void_p()
        t0 = time.perf_counter(); e = rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(mb << 20)); t1 = time.perf_counter()
        rt.cudaMemset(p, 0, ctypes.c_size_t(mb << 20)); rt.cudaDeviceSynchronize(); t2 = time.perf_counter()
        rt.cudaFree(p); t3 = time.perf_counter()
        res.append((mb, e, round((t1-t0)*1e3, 2), round((t2-t1)*1e3, 2), round((t3-t2)*1e3, 2)))
print(res)
