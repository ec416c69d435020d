"""Per-kv-tile event clocks of one attention CTA (profile build): the heaviest query tile
(blockIdx 0, tile T-1 of sequence 0 head 0).  Events per tile j: 0 softmax waits S_j,
1 S_j ready, 2 row max done, 3 P computed / waiting for O(j-1), 4 O(j-1) done, 5 P_j + rescale
published, 6 S_j MMAs issued, 7 O_j MMAs issued."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), "libfireq_prof.so"))
B, N, Hq, Hkv = [int(v) for v in sys.argv[1:5]] if len(sys.argv) > 4 else (1, 1024, 32, 8)
qb, kb, vb = synth.attention(B, N, Hq, Hkv, 5)
Q, K, V = (synth.bits_to_torch(x).cuda() for x in (qb, kb, vb))
cache = F.KVCache(K, V)
xq, beta = F.quantize_act(Q.reshape(B * Hq * N, 128))
q8, qs = xq.reshape(B, Hq, N, 128), beta.reshape(B, Hq, N)
for _ in range(3):
    F.kv4q8_attention(q8, qs, cache, Hq)
tr = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
F.debug_set_trace(tr)
F.kv4q8_attention(q8, qs, cache, Hq)
torch.cuda.synchronize()
F.debug_set_trace(None)
t = tr.cpu().numpy().reshape(64, 8).astype(np.int64)
T = N // 128
t0 = t[0, 0]
print("tile  wait_S  S_rdy  max_done  P_done  O(j-1)_done  published  S_issue  O_issue   (cycles from tile 0 softmax start)")
for j in range(T):
    print(f"{j:4d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in t[j]))
d = np.diff(t[:T, 5])
print("per-tile period (published -> published):", d.tolist())
