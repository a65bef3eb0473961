"""Repro probe for the host-vector PDL path: many calls of one shape with
fresh page-locked x each time, compared bit for bit with the device-tensor
call.  Prints failures per configuration."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1410_1726_b200 as kb
from oracle import naive

DT = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}

def pinned(a, shift=0):
    t = torch.empty(a.size + shift, dtype=DT[{np.float32: "s", np.float64: "d", np.complex64: "c", np.complex128: "z"}[a.dtype.type]], pin_memory=True)
    h = t.numpy()[shift:]; h[:] = a; return h

def run(tag, kind, d, op, shift, reps=200):
    rng = np.random.default_rng(1)
    ld = -(-d // 32) * 32
    t = torch.empty(ld * d, dtype=DT[tag], device="cuda")
    (torch.view_as_real(t) if tag in "cz" else t).uniform_(-1, 1)
    v = kb.MatrixView(t, d, d, ld, kb.precision(tag))
    fails = 0; first = None
    for r in range(reps):
        x = naive.fill(rng, d, tag); y = naive.fill(rng, d, tag)
        hx = pinned(x, shift)
        if kind == "symv":
            hv = kb.HermitianView(v, op)
            got = kb.symv_hemv(op, 1.0, hv, hx, 0.0, y).y_out
            want = kb.symv_hemv(op, 1.0, hv, torch.from_numpy(x).cuda(), 0.0, torch.from_numpy(y).cuda()).y_out.cpu().numpy()
        else:
            got = kb.gemv(op, 1.0, v, hx, 0.0, y).y_out
            want = kb.gemv(op, 1.0, v, torch.from_numpy(x).cuda(), 0.0, torch.from_numpy(y).cuda()).y_out.cpu().numpy()
        bad = np.nonzero(got != want)[0]
        if bad.size:
            fails += 1
            if first is None:
                first = (r, bad.size, bad[:3].tolist())
    print(tag, kind, d, op, "shift", shift, "fails", fails, "of", reps, "first", first, flush=True)

for tag in "sd":
    for shift in (0, 1):
        run(tag, "symv", 859, "l", shift)
run("s", "symv", 4096, "l", 1)
run("s", "gemv", 859, "n", 1)
run("d", "gemv", 4096, "t", 1)
