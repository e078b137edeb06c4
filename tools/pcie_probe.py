"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (sizes of the Llama 8K e2e step)."""
import torch, time
dev = torch.device("cuda")
h_in = torch.empty(100 * 2**20, dtype=torch.uint8).pin_memory()
h_out = torch.empty(64 * 2**20, dtype=torch.uint8).pin_memory()
d_in = torch.empty_like(h_in, device=dev)
d_out = torch.empty_like(h_out, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best
t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
t_both = timed(both)
def chunked():
    n = 8; c = h_in.numel() // n
    for i in range(n):
        with torch.cuda.stream(s1): d_in[i*c:(i+1)*c].copy_(h_in[i*c:(i+1)*c], non_blocking=True)
t_ch = timed(chunked)
print(f"H2D {h_in.numel()/t_h2d/1e9:.1f} GB/s  D2H {h_out.numel()/t_d2h/1e9:.1f} GB/s  "
      f"concurrent {(h_in.numel()+h_out.numel())/t_both/1e9:.1f} GB/s ({t_both*1e3:.2f} ms vs {1e3*(t_h2d+t_d2h):.2f} serial)  "
      f"H2D 8 chunks {h_in.numel()/t_ch/1e9:.1f} GB/s")
