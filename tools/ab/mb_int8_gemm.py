"""cuBLASLt int8 GEMM throughput (torch._int_mm) at heavy-Gram-like shapes:
the ceiling a tensor-core heavy walk would work against."""
import torch, time
for (M, K, N) in [(2048, 92160, 16384), (4096, 92160, 8192), (8192, 8192, 8192)]:
    a = torch.randint(0, 2, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(0, 127, (K, N), dtype=torch.int8, device="cuda").t().contiguous().t()
    torch._int_mm(a, b); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        torch._int_mm(a, b)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"int8 {M}x{K}x{N}: {ms:.2f} ms, {2*M*K*N/ms/1e9:.0f} TOPS")
