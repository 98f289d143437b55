"""PCIe copy costs for the e2e path: contiguous H2D / D2H vs 2-D (128-byte rows) D2H, pinned host."""
import torch, time
dev = torch.device("cuda")
def t(fn, reps=20):
    st = torch.cuda.current_stream(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); e1.synchronize()
    return e0.elapsed_time(e1) / reps
for mb in (4.7, 18.9, 6.3):
    n = int(mb * 1e6) // 2
    h = torch.empty(n, dtype=torch.float16).pin_memory(); d = torch.empty(n, dtype=torch.float16, device=dev)
    ms_h2d = t(lambda: d.copy_(h, non_blocking=True)); ms_d2h = t(lambda: h.copy_(d, non_blocking=True))
    print(f"{mb:5.1f} MB  H2D {ms_h2d*1e3:7.1f} us ({mb/ms_h2d:.1f} GB/s)   D2H {ms_d2h*1e3:7.1f} us ({mb/ms_d2h:.1f} GB/s)")
import ctypes
lib = ctypes.CDLL("libcudart.so") if False else None
h = torch.empty(96, 512, 64, dtype=torch.float16).pin_memory(); d = torch.empty(96, 512, 64, dtype=torch.float16, device=dev)
# strided (2-D) copy: same bytes as rows of 128 B via a transposed view trick
print("E-sized D2H contiguous", round(t(lambda: h.copy_(d, non_blocking=True)) * 1e3, 1), "us")
