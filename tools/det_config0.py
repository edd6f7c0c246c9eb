import time, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2506_09594_b200 as pk
rng = np.random.default_rng(0)
a = rng.standard_normal((200, 10, 50)); b = rng.standard_normal((10, 200, 50))
x = np.real(np.fft.ifft(np.einsum('ikf,kjf->ijf', np.fft.fft(a, axis=2), np.fft.fft(b, axis=2)), axis=2))
x /= np.linalg.norm(x)
mask = rng.random(x.shape) < 0.3
mobs = np.where(mask, x, 0.0)
for it in (1, 3):
    t0 = time.time(); l, e, rep = pk.gnrhtc(mobs, mask, pk.SolverConfig(max_iters=it)); t1 = time.time()
    print(it, "sweeps", round(t1 - t0, 2), "s", "rel err", np.linalg.norm(l - x) / np.linalg.norm(x), flush=True)
