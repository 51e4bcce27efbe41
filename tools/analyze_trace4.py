"""Summarise f2m_sweep_trace.bin written by the persistent sweep kernel (F2M_SWEEP_TRACE=first,count).

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
first, count, G, stride = np.frombuffer(raw[:16], np.int32)
G = -G  # header: (first, count, -columns, stride); v5 has one extra column: the master CTA
nt = count * G * 16
t = np.frombuffer(raw[16:16 + 8 * nt], np.uint64).astype(np.int64)[:count * G * stride].reshape(count, G, stride)
rest = np.frombuffer(raw[16 + 8 * nt:], np.int32)
master = None
if stride == 16:
    master = t[:, G - 1, 0].copy()
    t = t[:, :G - 1, :]
    G = G - 1
noff = rest[:G + 1]
nbr = rest[G + 1:G + 1 + noff[G]]
part = rest[G + 1 + noff[G]:]
if len(part) >= 4 * G + 2:
    lo, int_hi, nint, hoff = part[:G + 1], part[G + 1:2 * G + 1], part[2 * G + 1:3 * G + 1], part[3 * G + 1:4 * G + 2]
    own = (lo[1:] - lo[:-1]) * 32
    nbnd = own - (int_hi - lo[:-1]) * 32
    nh = hoff[1:] - hoff[:-1]
else:
    own = nbnd = nh = None
t0 = t[0, :, 0].min()
tt = np.where(t > 0, t - t0, 0)
names = ["top", "first_poll", "halo_staged", "bnd_start", "w0_interior", "barrier_B", "published", "bnd_published",
         "t0_rowdone", "t0_merged", "t0_reduced", "t0_decided"] + [f"ph{i}" for i in range(12, 16)]
print(f"sweeps {first}..{first + count - 1}, {G} CTAs, {noff[G]} CTA adjacencies "
      f"(mean {noff[G] / G:.1f} per CTA)")
cyc = np.diff(tt[:, :, 0], axis=0)
print(f"sweep period (top->top): median {np.median(cyc):.0f} ns, mean {cyc.mean():.0f}, p90 {np.percentile(cyc, 90):.0f}")
for ph in range(1, min(stride, 12)):
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
# per-CTA critical work after the halo: last boundary publish - halo staged (same sweep)
bw = np.median(np.where((tt[:, :, 7] > 0) & (tt[:, :, 2] > 0), tt[:, :, 7] - tt[:, :, 2], np.nan), axis=0)
print(f"per-CTA median (boundary published - halo staged): min {np.nanmin(bw):.0f} median {np.nanmedian(bw):.0f} "
      f"max {np.nanmax(bw):.0f} ns; worst CTAs {np.argsort(-np.nan_to_num(bw))[:5].tolist()}")
if own is not None:
    print(f"partition: own nodes median {np.median(own):.0f} max {own.max()}, boundary-phase rows median "
          f"{np.median(nbnd):.0f} max {nbnd.max()}, halo median {np.median(nh):.0f} max {nh.max()}, "
          f"neighbour CTAs max {np.diff(noff).max()}")
    for c in np.argsort(-np.nan_to_num(bw))[:6]:
        print(f"  CTA {c}: post-halo {bw[c]:.0f} ns, own {own[c]}, bnd rows {nbnd[c]}, halo {nh[c]}, "
              f"nbrs {noff[c + 1] - noff[c]}")
    print(f"  corr(post-halo, bnd rows) = {np.corrcoef(np.nan_to_num(bw), nbnd)[0, 1]:.2f}, "
          f"corr(post-halo, halo) = {np.corrcoef(np.nan_to_num(bw), nh)[0, 1]:.2f}")
lat_c = []
for c in range(G):
    nb = nbr[noff[c]:noff[c + 1]]
    if len(nb) == 0:
        lat_c.append(np.nan)
        continue
    prod = tt[:-1, nb, 7].max(axis=1)
    cons = tt[1:, c, 2]
    ok = (prod > 0) & (cons > 0)
    lat_c.append(np.median((cons - prod)[ok]) if ok.any() else np.nan)
lat_c = np.array(lat_c)
print(f"per-CTA median exchange latency: min {np.nanmin(lat_c):.0f} median {np.nanmedian(lat_c):.0f} "
      f"max {np.nanmax(lat_c):.0f} ns")
if stride == 16:
    for ph, nm in ((12, "bar->row loaded"), (13, "row scan"), (14, "publish"), (15, "bar->end")):
        v = t[:, :, ph]
        print(f"  warp0 {nm:16s}: median {np.median(v):6.0f} cycles  p90 {np.percentile(v, 90):6.0f}")
if master is not None and (master > 0).any():
    last_pub = t[:, :, 6].max(axis=1)
    ok = (master > 0) & (last_pub > 0)
    d = (master - last_pub)[ok]
    print(f"master: verdict k published - last CTA max(k) published: median {np.median(d):.0f} ns p90 {np.percentile(d, 90):.0f}")
    first_pub = np.where(t[:, :, 6] > 0, t[:, :, 6], np.iinfo(np.int64).max).min(axis=1)
    d2 = (last_pub - first_pub)[ok]
    print(f"        spread of max(k) publish times across CTAs: median {np.median(d2):.0f} ns")
    # when does a CTA need verdict k?  at the end of sweep k+7 (decision for k+8)
    need = t[7:, :, 11] if t.shape[0] > 7 else None
    if need is not None:
        wait = need - master[:-7, None]
        print(f"        decision(k+7) - verdict(k): median {np.median(wait):.0f} ns (negative = CTA waited)")
if own is not None:
    print("worst CTAs, per-phase medians relative to top (ns) and clock64 cycles:")
    for c in np.argsort(-np.nan_to_num(bw))[:4].tolist() + [int(np.argsort(np.nan_to_num(bw))[G // 2])]:
        ph = {names[p]: int(np.median(tt[:, c, p] - tt[:, c, 0])) for p in (2, 3, 4, 8, 7, 10, 11, 5, 6)}
        cyc = {k: int(np.median(t[:, c, p])) for k, p in (("rowload", 12), ("rowscan", 13), ("publish", 14), ("bar2end", 15))}
        spread = np.percentile(tt[:, c, 7] - tt[:, c, 2], [10, 50, 90]).astype(int).tolist()
        print(f"  CTA {c}: {ph} {cyc} post-halo p10/50/90 {spread}")
