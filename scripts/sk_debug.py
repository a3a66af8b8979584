import numpy as np, torch, sys, os
sys.path.insert(0, '.')
import paper_2402_10876_b200 as tw
from oracle import tilesparse_oracle as orc
k, n, m, g, s = 3072, 768, 8192, 128, 0.75
rng = np.random.default_rng(k + n + m)
w = tw.round_to(rng.normal(size=(k, n)).astype(np.float32))
a = tw.round_to(rng.normal(size=(m, k)).astype(np.float32))
plan, tsm = tw.prune_tw(w, s, g)
enc = tw.encode_cto(tsm)
ref = orc.c_gemm_cto_enc(a, enc)
# host model of the stream-K map (LPT order by K'*width)
kps = [(int(h) + 63) // 64 for h in enc.row_counts]
order = sorted(range(len(kps)), key=lambda i: -int(enc.row_counts[i]) * int(enc.col_counts[i]))
spm = sum(kps); T = (m // 128) * spm; P = min(148, T // max(kps))
print("kps", kps, "order", order, "spm", spm, "T", T, "P", P)
split_units = set()
off = {}; o = 0
for j in order: off[j] = o; o += kps[j]
for c in range(1, P):
    b = T * c // P
    mb = b // spm; rem = b % spm
    for j in order:
        if off[j] < rem < off[j] + kps[j]:
            split_units.add((mb, j))
print("split units", len(split_units))
for run in range(6):
    o = tw.gemm_tile_sparse(a, tsm).condensed.cpu().numpy()
    d = np.abs(o - ref) > 1e-4 * np.abs(ref).max()
    bad = set()
    for mb in range(m // 128):
        for j in range(3):
            if d[mb*128:(mb+1)*128, j*128:(j+1)*128].any(): bad.add((mb, j))
    print(run, "bad units", sorted(bad), "all split?", bad <= split_units)
