"""cuBLAS (torch.matmul, fp64) on the root-contraction GEMM shapes, for comparison with root_gemm_kernel."""
import torch, sys
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
for (F, B, R) in [(160000, 400, 100), (10000, 10000, 50)]:
    X = torch.randn(F, B, dtype=torch.float64, device=dev)
    Kb = torch.randn(B, R, dtype=torch.float64, device=dev)
    Kf = torch.randn(F, R, dtype=torch.float64, device=dev)
    for name, fn in (("NN  X@KRP_B", lambda: X @ Kb), ("TN  X^T@KRP_F", lambda: X.t() @ Kf)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): fn()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"F={F} B={B} R={R} {name}: {ms*1e3:.1f} us  {2*F*B*R/ms/1e9:.2f} TFLOP/s")
