import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_1410_1726_b200 as kb
from oracle import naive
from test_gpu_hostvec import pinned, dev_view, DT

tag = "d"
for kind in ["pinned", "pinned_shifted", "pageable"]:
    for uplo in "lu":
        rng = np.random.default_rng(102)
        for d, beta in [(4096, 0.0), (1001, 0.5), (12288, 0.0)]:
            v, a = dev_view(rng, d, d, tag, host=False)
            hv = kb.HermitianView(v, uplo)
            x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
            if kind == "pinned":
                hx, hy = pinned(x), pinned(y)
            elif kind == "pinned_shifted":
                hx, hy = pinned(x, 1), pinned(y, 1)
            else:
                hx, hy = x.copy(), y.copy()
            got = kb.symv_hemv(uplo, 1.5, hv, hx, beta, hy).y_out
            got_copy = np.array(got)
            want = kb.symv_hemv(uplo, 1.5, hv, torch.from_numpy(x).cuda(), beta, torch.from_numpy(y).cuda()).y_out.cpu().numpy()
            got2 = np.array(kb.symv_hemv(uplo, 1.5, hv, hx, beta, hy).y_out)
            if d <= 4096:
                host = v.data.cpu().numpy()
                A = naive.window(host, v.ld, d, d)
                ref = naive.naive_symv_hemv(1.5, np.array(A), uplo, x, beta, y, False)
                e_got, e_want = float(np.max(np.abs(got_copy - ref))), float(np.max(np.abs(want - ref)))
            else:
                e_got = e_want = None
            nbad = int(np.sum(got_copy != want)); nbad_after = int(np.sum(got != got_copy)); nbad2 = int(np.sum(got2 != want))
            print(kind, uplo, d, beta, "bad", nbad, "changed_after", nbad_after, "repeat_bad", nbad2,
                  "err got", e_got, "err want", e_want, "x ok", np.array_equal(hx, x), "y ok", np.array_equal(hy, y), flush=True)
