"""Summarise f2m_sweep_trace.bin written by the v4 sweep kernel (F2M_SWEEP_TRACE=first,count).

phases (globaltimer ns per sweep, CTA): 0 top (after barrier A) | 1 first halo poll returned |
2 halo staged | 3 boundary compute starts | 4 warp 0 interior done | 5 after barrier B |
6 max published | 7 last boundary value published.
The file ends with the CTA adjacency (nbr_off[G+1], nbr[...]), so the exchange latency can be
measured edge by edge: halo staged (consumer, sweep s) - last boundary publish of its slowest
neighbour (producer, sweep s-1)."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "f2m_sweep_trace.bin"
raw = open(path, "rb").read()
first, count, G = np.frombuffer(raw[:12], np.int32)
nt = count * G * 8
t = np.frombuffer(raw[12:12 + 8 * nt], np.uint64).astype(np.int64).reshape(count, G, 8)
rest = np.frombuffer(raw[12 + 8 * nt:], np.int32)
noff = rest[:G + 1]
nbr = rest[G + 1:G + 1 + noff[G]]
t0 = t[0, :, 0].min()
tt = np.where(t > 0, t - t0, 0)
names = ["top", "first_poll", "halo_staged", "bnd_start", "w0_interior", "barrier_B", "published", "bnd_published"]
print(f"sweeps {first}..{first + count - 1}, {G} CTAs, {noff[G]} CTA adjacencies "
      f"(mean {noff[G] / G:.1f} per CTA)")
cyc = np.diff(tt[:, :, 0], axis=0)
print(f"sweep period (top->top): median {np.median(cyc):.0f} ns, mean {cyc.mean():.0f}, p90 {np.percentile(cyc, 90):.0f}")
for ph in range(1, 8):
    valid = t[:, :, ph] > 0
    if not valid.any():
        continue
    d = (tt[:, :, ph] - tt[:, :, 0])[valid]
    print(f"  top -> {names[ph]:14s}: median {np.median(d):7.0f} ns  p10 {np.percentile(d, 10):7.0f}  "
          f"p90 {np.percentile(d, 90):7.0f}")
# exchange latency: consumer halo staged at s vs slowest neighbour's boundary publish at s-1
lat, wait = [], []
for c in range(G):
    nb = nbr[noff[c]:noff[c + 1]]
    if len(nb) == 0:
        continue
    prod = tt[:-1, nb, 7].max(axis=1)          # sweep s-1
    cons = tt[1:, c, 2]                        # sweep s
    top = tt[1:, c, 0]
    ok = (prod > 0) & (cons > 0)
    lat.append((cons - prod)[ok])
    wait.append((prod - top)[ok])
lat = np.concatenate(lat)
wait = np.concatenate(wait)
print(f"exchange: halo staged - slowest neighbour's last boundary publish: median {np.median(lat):.0f} ns "
      f"p10 {np.percentile(lat, 10):.0f} p90 {np.percentile(lat, 90):.0f}")
print(f"          slowest neighbour's publish - own top: median {np.median(wait):.0f} ns "
      f"(>0: this CTA waits for its neighbours)")
sk = tt[:, :, 0].max(1) - tt[:, :, 0].min(1)
print(f"CTA skew at top: median {np.median(sk):.0f} ns max {sk.max():.0f}")
