"""Per-block timeline of one CTA of K5 at HY (needs a -DDFS_ATTN_TRACE_BUILD library via DFS_B200_LIB)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['DFS_ATTN_TRACE'] = 'gpurun_out/attn_trace.bin'
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
from bench import smooth_fields
dims, H, d = (33, 45, 80), 24, 128
n = 33 * 45 * 80
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
perm = m.hilbert3d_order(dims)
qh, pq = ops.permute_to_hnd(q, perm, 16); kh, pk = ops.permute_to_hnd(k, perm, 16); vh, _ = ops.permute_to_hnd(v, perm, 0)
S = ops.score_pooled(pq, pk, n, m.ScoringParams(128, 16)); lut = m.topk_lut(S, 0.1); ptr = ops.lut_row_ptr(H, 929, 93)
os.makedirs('gpurun_out', exist_ok=True)
o = m.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), 128); torch.cuda.synchronize()
t = np.fromfile('gpurun_out/attn_trace.bin', dtype=np.uint64).reshape(40, 256).astype(np.int64)
names = ['kv_wait_start', 'kv_wait_done', 'p_wait_start', 'p_wait_done', 'A_s_wait', 'A_s_ready', 'A_barrier',
         'A_arrive', 'B_s_wait', 'B_s_ready', 'B_barrier', 'B_arrive']
lo, hi = 60, 120
t0 = t[0, lo * 2]
for i, nm in enumerate(names):
    print(f"{nm:14s}", ' '.join(f"{x - t0:7d}" for x in t[i, lo:lo + 12]))
for s, base in (("A", 4), ("B", 8)):
    w = (t[base + 1, lo:hi] - t[base, lo:hi]).mean()
    busy = (t[base + 3, lo:hi] - t[base + 1, lo:hi]).mean()
    pre = (t[base + 2, lo:hi] - t[base + 1, lo:hi]).mean()
    per = np.diff(t[base + 3, lo:hi]).mean()
    print(f"stream {s}: period/block {per:.0f} (2 blocks of the tile), S wait {w:.0f}, busy {busy:.0f} (to barrier {pre:.0f})")
# row-split softmax phases of the two warps sharing SMSP 2 (warp 2: rows 64-79, warp 6: rows 80-95):
# s_wait -> S ready -> S loaded -> exponentials done -> P stored -> next block
for nm, (w0, w1, ld, ex, st) in (("warp 2", (4, 5, 12, 14, 7)), ("warp 6", (8, 9, 13, 15, 11))):
    seg = [("S wait", w0, w1), ("TMEM ld", w1, ld), ("exp loop", ld, ex), ("P store", ex, st)]
    out = [f"{n} {(t[b, lo:hi] - t[a, lo:hi]).mean():6.0f}" for n, a, b in seg]
    out.append(f"to next {(t[w0, lo + 1:hi + 1] - t[st, lo:hi]).mean():6.0f}")
    out.append(f"period {np.diff(t[st, lo:hi]).mean():6.0f}")
    print(f"  {nm}: " + " | ".join(out))
print("  warp 6 ahead of warp 2 by (S ready):", (t[5, lo:hi] - t[9, lo:hi]).mean())
# MMA chain: last P_j in (p_wait_done) -> PV_j issued (16) -> QK_{j+2} issued (17, index j+2) -> S_{j+2} seen (5, j+2)
j = np.arange(lo, hi - 2)
print(f"  MMA chain: P_j seen -> PV_j issued {(t[16, j] - t[3, j]).mean():6.0f} | -> QK_j+2 issued {(t[17, j + 2] - t[16, j]).mean():6.0f}"
      f" | QK issued -> S_j+2 seen by warp 2 {(t[5, j + 2] - t[17, j + 2]).mean():6.0f}"
      f" | P_j arrive(warp 2) -> S_j+2 seen {(t[5, j + 2] - t[7, j]).mean():6.0f}")
pw = (t[3, lo:hi] - t[2, lo:hi]).mean()
kvw = (t[1, 2 * lo:2 * hi] - t[0, 2 * lo:2 * hi]).mean()
print(f"MMA: p_full wait/PV {pw:.0f}, kv wait/ring entry {kvw:.0f}, PV period {np.diff(t[2, lo:hi]).mean():.0f}")
# raw per-block timeline (cycles relative to warp 2's S_j ready)
print("  j | S_j rdy(w2) | P_j arr(w2) | P_j seen(MMA) | PV_j issued | QK_j issued | kv waits (K,V entries)")
for jj in range(lo, lo + 6):
    b = t[5, jj]
    print(f"  {jj} | 0 | {t[7, jj] - b} | {t[3, jj] - b} | {t[16, jj] - b} | {t[17, jj] - b} |"
          f" {[int(t[1, e] - t[0, e]) for e in range(2 * jj, 2 * jj + 2)]}")

arr = np.stack([t[18 + w, lo:hi] for w in range(8)])  # warps 1..8
first = arr.min(0)
print("  P_j arrival after the first warp's, per softmax warp 1..8 (SMSP = warp % 4):",
      " ".join(f"w{w + 1}:{(arr[w] - first).mean():.0f}" for w in range(8)))
print("  last warp's arrival -> P_j seen by MMA:", (t[3, lo:hi] - arr.max(0)).mean())
seen = np.stack([t[26 + w, lo:hi] for w in range(8)])
print("  per softmax warp 1..8: S_j seen after the first warp's | busy S seen -> P arrive:")
print("   ", " ".join(f"w{w + 1}:{(seen[w] - seen.min(0)).mean():.0f}|{(arr[w] - seen[w]).mean():.0f}" for w in range(8)))
