import ctypes, glob, torch
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*")
rt = ctypes.CDLL(libs[0])
v = ctypes.c_size_t()
print("get rc", rt.cudaDeviceGetLimit(ctypes.byref(v), 5), "granularity", v.value, flush=True)
n = 1 << 27
x = torch.rand(n, dtype=torch.float64, device="cuda")
for g in (128, 32):
    print("set rc", rt.cudaDeviceSetLimit(5, ctypes.c_size_t(g)), flush=True)
    rt.cudaDeviceGetLimit(ctypes.byref(v), 5); print("granularity now", v.value, flush=True)
    a = x.view(-1, 8)[:, :4].contiguous()
    b = x.view(-1, 16)[:, :4].contiguous()
    torch.cuda.synchronize()
print("done")
