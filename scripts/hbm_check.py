"""HBM copy-bandwidth sanity check (torch copy_, the MEASURED_PEAKS.json recipe) at a few sizes."""
import torch

torch.cuda.set_device(0)
for n_bytes in (1 << 30, 2 << 30, 4 << 30):
    for dt in (torch.bfloat16, torch.float64):
        n = n_bytes // torch.tensor([], dtype=dt).element_size()
        a = torch.randn(n, device="cuda").to(dt) if dt != torch.float64 else torch.randn(n, device="cuda", dtype=dt)
        b = torch.empty_like(a)
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"copy {n_bytes >> 20} MiB {dt}: {2 * n_bytes / (best * 1e-3) / 1e9:.1f} GB/s", flush=True)
        del a, b
