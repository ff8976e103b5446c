"""C2-sized AA window (N = 5e7 fp32, m = 10): time push / weights / step
separately with CUDA events (for ncu: kernels k_aa_push / k_aa_step)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2008_11778_b200 import anderson
    n = 50_000_000
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    vecs = [(torch.randn(n, generator=g, device=dev), torch.randn(n, generator=g, device=dev))
            for _ in range(m + 6)]
    win = anderson.AAWindow(n, m, dtype="float32", device=dev)
    out = torch.empty(n, device=dev)
    for k in range(m + 1):
        win.push(*vecs[k])
    tp, tw, ts = [], [], []
    for k in range(m + 1, m + 6):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        win.push(*vecs[k])
        e[1].record()
        t0 = time.perf_counter()
        w = anderson.aa_weights(win)
        tw.append((time.perf_counter() - t0) * 1e3)
        e[2].record()
        anderson.aa_step(win, weights=w, out=out)
        e3 = torch.cuda.Event(enable_timing=True)
        e3.record()
        torch.cuda.synchronize()
        tp.append(e[0].elapsed_time(e[1]))
        ts.append(e[2].elapsed_time(e3))
    gbs = lambda nb, ms: nb / (ms / 1e3) / 1e9
    pm, sm = min(tp), min(ts)
    print(f"push {pm:.3f} ms ({gbs((m + 8) * n * 4, pm):.0f} GB/s of {(m + 8) * n * 4 / 1e9:.1f} GB), "
          f"weights(host) {min(tw):.3f} ms, step {sm:.3f} ms ({gbs((m + 2) * n * 4, sm):.0f} GB/s)")


if __name__ == "__main__":
    main()
