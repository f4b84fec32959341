"""Dev aid: cost of cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize)."""
import ctypes, time, glob, os
import torch
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
       glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(libs[0])
LIM = 0x06  # cudaLimitPersistingL2CacheSize
maxp = ctypes.c_int()
rt.cudaDeviceGetAttribute(ctypes.byref(maxp), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
print("max persisting", maxp.value, "lib", libs[0])
def t(v, what):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); r = rt.cudaDeviceSetLimit(LIM, ctypes.c_size_t(v)); dt = time.perf_counter() - t0
    print(f"{what}: set {v} -> rc {r}, {1e3*dt:.2f} ms")
t(maxp.value, "raise"); t(maxp.value, "raise again"); t(0, "lower"); t(maxp.value, "raise")
x = torch.empty(40 << 30, dtype=torch.uint8, device="cuda"); x.fill_(1); torch.cuda.synchronize()
t(0, "lower (40 GB allocated)"); t(maxp.value, "raise (40 GB allocated)")
x.fill_(2)
t(0, "lower (busy)"); t(maxp.value, "raise (after busy)")
