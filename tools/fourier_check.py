import os, sys, json, math
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_11629_b200 as R
from paper_1811_11629_b200 import bitsource, stats
g = json.load(open("tests/golden/battery.json"))
plist = bitsource.interstream_params(R.DEFAULT_MASTER_SEED, g["streams"][0], len(g["streams"]))
make = lambda: bitsource.BitSource([R.init_vector(p, m0=0, s0=1, mv=g["lanes"]) for p in plist], "float_leading")
rep = stats.fourier_test(make(), g["budget"])
want = next(r for r in g["reports"] if r["name"] == "fourier")
print("gpu", rep.result.statistic, rep.result.p_value, "golden", want["statistic"], want["p"])
m = stats.FOURIER_M; blocks = g["budget"] // (2 * m)
zt = make().take(blocks * 2 * m).view(blocks, 2 * m)
cg = (torch.fft.fft(torch.complex(zt[:, 0::2] - 0.5, zt[:, 1::2] - 0.5), dim=-1) / math.sqrt(m)).cpu().numpy()
z = zt.cpu().numpy()
cn = np.fft.fft((z[:, 0::2] - 0.5) + 1j * (z[:, 1::2] - 0.5), axis=-1) / math.sqrt(m)
print("max diff", np.abs(cg - cn).max())
edges = stats._normal_edges()
for a, b in ((cg.real, cn.real), (cg.imag, cn.imag)):
    ia, ib = np.searchsorted(edges, a.reshape(-1)), np.searchsorted(edges, b.reshape(-1))
    bad = np.flatnonzero(ia != ib)
    print("moved", bad.size, [(float(b.reshape(-1)[k]), float(np.min(np.abs(edges - b.reshape(-1)[k])))) for k in bad[:5]])
