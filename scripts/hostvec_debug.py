import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1410_1726_b200 as kb
from oracle import naive

def pinned(a, shift=0):
    t = torch.empty(a.size + shift, dtype=torch.float64, pin_memory=True)
    h = t.numpy()[shift:]; h[:] = a; return h

rng = np.random.default_rng(5)
for d in (1001, 4096):
    buf = np.zeros(d * d); win = naive.window(buf, d, d, d); win[:, :] = naive.fill(rng, (d, d), "d")
    v = kb.MatrixView(torch.from_numpy(buf).cuda(), d, d, d, kb.precision("d")); a = np.array(win)
    hv = kb.HermitianView(v, "l")
    x, y = naive.fill(rng, d, "d"), naive.fill(rng, d, "d")
    ref = naive.naive_symv_hemv(1.5, a, "l", x, 0.5, y, False)
    want = kb.symv_hemv("l", 1.5, hv, torch.from_numpy(x).cuda(), 0.5, torch.from_numpy(y).cuda()).y_out.cpu().numpy()
    for name, hx, hy in [("aligned", pinned(x), pinned(y)), ("x shifted", pinned(x, 1), pinned(y)),
                         ("y shifted", pinned(x), pinned(y, 1)), ("both shifted", pinned(x, 1), pinned(y, 1)),
                         ("pageable", x.copy(), y.copy())]:
        errs = []
        for rep in range(3):
            got = kb.symv_hemv("l", 1.5, hv, hx, 0.5, hy).y_out
            bad = np.nonzero(got != want)[0]
            errs.append((len(bad), bad[:3].tolist(), float(np.max(np.abs(got - ref))) if ref is not None else None))
        print(d, name, errs, flush=True)
    print("want vs ref", float(np.max(np.abs(want - ref))) if ref is not None else None)
