"""Writes SYMV/HEMV results of a fixed set of cases to an .npz (run it under
KBLAS_SYMV_EPILOGUE=32 and without, then compare: the 128-row epilogue
must give bit-identical y).  Cases: single GPU wide-kernel orders (L/U,
S/D/C/Z, beta 0 / -0.5, a misaligned diagonal offset) and the mgpu API
with nb = 128 / 256 / 64 on 2-3 logical GPUs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1410_1726_b200 as kb

out = {}
DT = {"s": torch.float32, "d": torch.float64, "c": torch.complex64, "z": torch.complex128}
g = torch.Generator(device="cuda").manual_seed(7)
for tag in "sdcz":
    for d in (13000, 20001):
        ld = -(-d // 32) * 32 + 32
        t = torch.empty(ld * (d + 5), dtype=DT[tag], device="cuda")
        (torch.view_as_real(t) if tag in "cz" else t).uniform_(-1, 1, generator=g)
        v = kb.MatrixView(t, d, d, ld, kb.precision(tag))
        x = torch.empty(d, dtype=DT[tag], device="cuda"); (torch.view_as_real(x) if tag in "cz" else x).uniform_(-1, 1, generator=g)
        y = torch.empty(d, dtype=DT[tag], device="cuda"); (torch.view_as_real(y) if tag in "cz" else y).uniform_(-1, 1, generator=g)
        herm = tag in "cz"
        for uplo in "lu":
            hv = kb.HermitianView(v, uplo)
            for beta in (0.0, -0.5):
                out[f"{tag}{d}{uplo}{beta}"] = kb.symv_hemv(uplo, 1.25, hv, x, beta, y, hermitian=herm).y_out.cpu().numpy()
            # misaligned diagonal offset (lead rows)
            pv = kb.MatrixView(t, d + 5, d + 5, ld, kb.precision(tag))
            out[f"{tag}{d}{uplo}off"] = kb.symv_hemv_offset(uplo, 0.5, kb.HermitianView(pv, uplo), 3, d, x, 0.25, y,
                                                            hermitian=herm).y_out.cpu().numpy()
        for nb, G in ((128, 2), (256, 3), (64, 2)):
            dm = kb.distribute(v, nb, G)
            for uplo in "lu":
                out[f"{tag}{d}mgpu{nb}{G}{uplo}"] = kb.symv_hemv_mgpu(uplo, 0.75, dm, x, 0.5, y, kb.KernelConfig(nb, 2),
                                                                       hermitian=herm)[0].y_out.cpu().numpy()
            del dm
np.savez(sys.argv[1], **out)
print("wrote", len(out), "cases")
