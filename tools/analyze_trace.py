"""Summarise f2m_sweep_trace.bin (F2M_SWEEP_TRACE=first,count): per-phase latencies of the v3 sweep kernel.
phases: 0 top (after barrier A) | 1 neighbours ready | 2 halo staged | 3 helper done | 4 warp0 interior done |
        5 after barrier B | 6 published"""
import sys
import numpy as np
path = sys.argv[1] if len(sys.argv) > 1 else "f2m_sweep_trace.bin"
with open(path, "rb") as f:
    first, count, G = np.frombuffer(f.read(12), np.int32)
    t = np.frombuffer(f.read(), np.uint64).astype(np.int64).reshape(count, G, 8)
t = t - t[0, :, 0].min()
names = ["top", "nbr_ready", "halo_staged", "bnd_start", "w0_interior", "barrier_B", "published", "last_warp_done"]
print(f"sweeps {first}..{first+count-1}, {G} CTAs")
cyc = np.diff(t[:, :, 0], axis=0)
print(f"sweep period (top->top): median {np.median(cyc):.0f} ns, mean {cyc.mean():.0f}, p90 {np.percentile(cyc,90):.0f}")
for ph in range(1, 8):
    d = t[:, :, ph] - t[:, :, 0]
    if (t[:, :, ph] <= 0).all() or np.abs(d).max() > 1e9:
        continue
    print(f"  top -> {names[ph]:12s}: median {np.median(d):7.0f} ns  p90 {np.percentile(d,90):7.0f}  max {d.max():7.0f}")
d = t[1:, :, 0] - t[:-1, :, 6]
print(f"  published -> next top: median {np.median(d):7.0f} ns p90 {np.percentile(d,90):7.0f}")
# skew across CTAs
sk = t[:, :, 0].max(1) - t[:, :, 0].min(1)
print(f"CTA skew at top: median {np.median(sk):.0f} ns max {sk.max():.0f}")
