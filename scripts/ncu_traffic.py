#!/usr/bin/env python
"""DRAM byte evidence for every variant (run on the GPU box under ncu).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --kernel-name regex:kblas_ --csv --log-file gpurun_out/traffic.csv \
        python scripts/ncu_traffic.py run > gpurun_out/traffic_seq.jsonl
    python scripts/ncu_traffic.py parse gpurun_out/traffic.csv gpurun_out/traffic_seq.jsonl   (here)

`run` calls every --op of bench.py (S/D/C/Z GEMV-N/T/C, SYMV/HEMV-L/U) at
N = 32768 and 60000 with ld = N, the configs[3] offset kernels on a
16384^2 parent, and the configs[4] per-GPU partial at N = 100000 (G = 1,
nb = 128), once each, and prints one JSON line per call with the number of
library kernels it launched (the launches are consumed in order when
parsing).  `parse` writes profiles/traffic.json (dominant kernel's DRAM
read + write bytes per launch, read by bench.py as roofline.traffic) and
profiles/r2_traffic_table.md (traffic / algorithmic bytes, flagged above
1.02).
"""

from __future__ import annotations

import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = (32768, 60000)
OFFSETS = ((1, 1), (7, 3), (13, 13))


def run():
    import torch

    from bench import OPS, alg_bytes
    from paper_1410_1726_b200 import _lib, roofline
    from paper_1410_1726_b200.core import precision
    from paper_1410_1726_b200.multidevice import partial_mv

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev).cuda_stream

    only = [k for k in os.environ.get("KEYS", "").split(",") if k]

    def emit(key, fn, nbytes, plan_hint=""):
        if only and key not in only:
            return
        fn()  # warm (tile tables, workspace): not counted
        torch.cuda.synchronize()
        l0 = _lib.launch_count()
        fn()
        torch.cuda.synchronize()
        print(json.dumps({"key": key, "warm_launches": None, "launches": _lib.launch_count() - l0,
                          "alg_bytes": int(nbytes), "plan": _lib.last_plan()}), flush=True)

    def gen(p, n_elems):
        t = torch.empty(n_elems, dtype=p.torch_dtype, device=dev)
        (torch.view_as_real(t) if p.is_complex else t).uniform_(-1, 1)
        return t

    by_prec = {}
    for name, (tag, family, op, herm) in OPS.items():
        by_prec.setdefault(tag, []).append(name)
    def want(kind):
        return not only or any(k.startswith(kind) == (kind != "") for k in only) if kind else (
            not only or any(not k.startswith(("offset_", "mgpu_")) for k in only))

    for n in SIZES if want("") else ():
        for tag in "sdcz":
            p = precision(tag)
            A = gen(p, n * n)
            x, y = gen(p, n), gen(p, n)
            one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
            for name in by_prec[tag]:
                _, family, op, herm = OPS[name]
                if family == "symv":
                    rname = {("s", False): "ssymv", ("d", False): "dsymv", ("c", True): "chemv",
                             ("z", True): "zhemv"}[(tag, herm)]
                    f = getattr(lib, f"kblas_{rname}_async")
                    call = (lambda f=f, op=op: f(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero,
                                                 y.data_ptr(), 1, st))
                else:
                    f = getattr(lib, f"kblas_{tag}gemv_async")
                    call = (lambda f=f, op=op: f(op.encode(), n, n, one, A.data_ptr(), n, x.data_ptr(), 1, zero,
                                                 y.data_ptr(), 1, st))

                def fn(call=call):
                    assert call() == 0

                emit(f"{name}_{n}", fn, alg_bytes(tag, family, n, n, op))
            del A
            torch.cuda.empty_cache()
    # configs[3]: offset kernels on a 16384^2 parent (true-submatrix bytes)
    N = 16384
    for tag in "sdcz" if want("offset_") else ():
        p = precision(tag)
        A = gen(p, N * N)
        x, y = gen(p, N), gen(p, N)
        one, zero = _lib.scalar(tag, 1.0), _lib.scalar(tag, 0.0)
        for (i, j) in OFFSETS:
            sm, sn = N - i, N - j
            for trans in "nt":
                f = getattr(lib, f"kblas_{tag}gemv_offset_async")

                def fn(f=f, trans=trans, i=i, j=j, sm=sm, sn=sn):
                    assert f(trans.encode(), sm, sn, one, A.data_ptr(), N, x.data_ptr(), 1, zero, y.data_ptr(), 1,
                             i, j, st) == 0

                emit(f"offset_{tag}gemv_{trans}_{i}_{j}", fn, roofline.gemv_bytes(p, sm, sn, trans))
            if i == j:
                rname = {"s": "ssymv", "d": "dsymv", "c": "chemv", "z": "zhemv"}[tag]
                f = getattr(lib, f"kblas_{rname}_offset_async")
                for uplo in "lu":
                    def fn(f=f, uplo=uplo, i=i):
                        assert f(uplo.encode(), N - i, one, A.data_ptr(), N, x.data_ptr(), 1, zero, y.data_ptr(), 1,
                                 i, st) == 0

                    emit(f"offset_{rname}_{uplo}_{i}_{i}", fn, roofline.symv_bytes(p, N - i))
        del A
        torch.cuda.empty_cache()
    # configs[4]: the per-GPU partial at N = 100000, G = 1, nb = 128
    from paper_1410_1726_b200.core import MatrixView

    n, nb = 100000, 128
    for tag, herm in (("d", False), ("z", True)) if want("mgpu_") else ():
        p = precision(tag)
        A = gen(p, n * n)
        v = MatrixView(A, n, n, n, p)
        x, out = gen(p, n), gen(p, n)

        def fn(v=v, x=x, out=out, p=p, herm=herm):
            partial_mv(p, "s", "l", n, n, 1.0, v, x, out, 1, 0, nb, herm)

        emit(f"mgpu_{'dsymv' if tag == 'd' else 'zhemv'}_{n}_G1", fn, roofline.symv_bytes(p, n))
        del A, v, fn, x, out
        torch.cuda.empty_cache()


def parse(csv_path, seq_path):
    with open(csv_path) as fh:
        text = fh.read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    # one row per (launch, metric)
    launches = {}
    order = []
    for r in rows:
        lid = int(r["ID"])
        if lid not in launches:
            launches[lid] = {"name": r["Kernel Name"]}
            order.append(lid)
        val = float(str(r["Metric Value"]).replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
                 "msecond": 1e-3, "second": 1}.get(unit, 1)
        launches[lid][r["Metric Name"]] = val * scale
    seq = [json.loads(line) for line in open(seq_path) if line.strip().startswith("{")]
    # every key is called twice (warm + measured); consume in order
    it = iter(order)
    table = []
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for ent in seq:
        for _ in range(ent["launches"]):  # warm call
            next(it)
        ks = [launches[next(it)] for _ in range(ent["launches"])]
        main = max(ks, key=lambda k: k.get("gpu__time_duration.sum", 0))
        b = main.get("dram__bytes_read.sum", 0) + main.get("dram__bytes_write.sum", 0)
        tot = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
        t = main.get("gpu__time_duration.sum", 0)
        traffic[ent["key"]] = int(b)
        table.append((ent["key"], main["name"].split("(")[0].split("<")[0].replace("void ", ""), ent["alg_bytes"], b,
                      tot, t, ent["plan"]))
    with open(tpath, "w") as fh:
        json.dump(dict(sorted(traffic.items())), fh, indent=1)
    lines = ["# DRAM traffic per variant (ncu, cold caches, one launch at a time)", "",
             "`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none`"
             " over `scripts/ncu_traffic.py run` (one B200). Algorithmic bytes: SURVEY §8(d) (true submatrix only).",
             "Main = the streaming kernel; ratio = its DRAM read+write / algorithmic bytes; all = every library "
             "kernel of the call (epilogue included). Ratios above 1.02 are flagged.", "",
             "| variant | main kernel | algorithmic GB | main DRAM GB | ratio | call DRAM GB | call ratio | main us | main GB/s (cold) |",
             "|---|---|---|---|---|---|---|---|---|"]
    for key, name, alg, b, tot, t, plan in table:
        r, rt = b / alg, tot / alg
        flag = " **>1.02**" if r > 1.02 else ""
        lines.append(f"| {key} | {name} | {alg / 1e9:.4f} | {b / 1e9:.4f} | {r:.4f}{flag} | {tot / 1e9:.4f} | "
                     f"{rt:.4f} | {t * 1e6:.1f} | {alg / t / 1e9 if t else 0:.0f} |")
    out = os.path.join(ROOT, "profiles", "r2_traffic_table.md")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2], sys.argv[3])
