import time, torch, sys
sys.path.insert(0, "/root/repo")
import paper_2305_16513_b200 as ss
x = torch.randn(64, 1 << 20, device="cuda")
xi = torch.randint(-1000, 1000, (1 << 26,), device="cuda", dtype=torch.int32)
y = torch.empty(64, (1 << 20) - 2, device="cuda")
yi = torch.empty((1 << 26) - 2, device="cuda", dtype=torch.int32)
s = torch.cuda.current_stream().cuda_stream
f = [0.1, 0.2, 0.3]
def t(fn, n=200):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n): fn()
    b = time.perf_counter()
    torch.cuda.synchronize()
    c = time.perf_counter()
    return (b - a) / n * 1e6, (c - a) / n * 1e6
print("ss_pool_sum i32 (raw ctypes): host %.1f us/call, total %.1f" % t(lambda: ss.ss_pool_sum(xi.data_ptr(), yi.data_ptr(), 1 << 26, 1, 3, 1, ss.SS_I32, s)))
print("ss_conv1d f32 k3 (raw):        host %.1f us/call, total %.1f" % t(lambda: ss.ss_conv1d(x.data_ptr(), y.data_ptr(), 1 << 20, 64, f, 3, 1, ss.SS_F32, s)))
print("torch Event create+record:     host %.1f us" % t(lambda: torch.cuda.Event(enable_timing=True).record())[0])
