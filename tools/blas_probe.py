"""Measure cuBLAS FP64 ceilings on this GPU (DGEMM and ZGEMM via torch.matmul)."""
import torch, json
def t(dtype, n, reps=5):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f = (8 if dtype.is_complex else 2) * n ** 3
    return f / (ms * 1e-3) / 1e12, ms
out = {}
for dt, n in [(torch.float64, 8192), (torch.complex128, 4096), (torch.complex128, 8192), (torch.complex128, 512), (torch.complex128, 256)]:
    tf, ms = t(dt, n)
    out[f"{dt}_{n}"] = {"tflops": tf, "ms": ms}
    print(dt, n, f"{tf:.2f} TFLOP/s {ms:.3f} ms", flush=True)
# batched small zgemm
for n, bs in [(128, 1024), (256, 256)]:
    a = torch.randn(bs, n, n, dtype=torch.complex128, device="cuda"); b = torch.randn(bs, n, n, dtype=torch.complex128, device="cuda")
    for _ in range(2): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("batched zgemm", n, bs, f"{8*bs*n**3/(ms*1e-3)/1e12:.2f} TFLOP/s")
json.dump(out, open("gpurun_out/blas_probe.json", "w"), indent=1)
