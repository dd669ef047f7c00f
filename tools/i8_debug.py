"""Debug: whole-data shifted Gram of the int8 path vs numpy, per 64x64 tile."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_13185_b200 import plan as P

n, k, m, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rng = np.random.default_rng(3)
x = rng.uniform(-5, 5, k) + rng.uniform(0.5, 2, k) * rng.standard_normal((n, k))
y = rng.standard_normal((n, m)) + 3
labels = (rng.permutation(n) % p + 1).astype(np.int32)
if len(sys.argv) > 5 and sys.argv[5] == "contig":
    labels = (np.arange(n) * p // n + 1).astype(np.int32)
dev = torch.device("cuda", 0)
tx, ty, tl = (torch.from_numpy(a).to(dev) for a in (x, y, labels))
pl = P.DevicePlan(n, k, m, p)
pl.bind_labels(tl, True)
pl.gram(tx, ty)
kp = int(round(pl.partial_count ** 0.5))
g = torch.empty(pl.partial_count, dtype=torch.float64, device=dev)
pl.partial_into(g)
torch.cuda.synchronize()
g = g.view(kp, kp).cpu().numpy()
z = np.zeros((n, kp))
z[:, :k] = x - x[0]
z[:, k:k + m] = y - y[0]
z[:, k + m] = 1
ref = z.T @ z
d = np.sqrt(np.abs(np.diag(ref))) + 1e-300
err = np.abs(g - ref) / np.outer(d, d)
nt = kp // 64
for i in range(nt):
    print(" ".join(f"{err[64*i:64*i+64, 64*j:64*j+64].max():8.1e}" if j >= i else "   -    " for j in range(nt)))
bad = np.argwhere(np.triu(err) > 1e-10)
print("bad entries", len(bad), bad[:10].tolist(), "rows", sorted(set(bad[:, 0].tolist()))[:20], "cols", sorted(set(bad[:, 1].tolist()))[:20])
