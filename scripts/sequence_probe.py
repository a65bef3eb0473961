"""Per-call time of SYMV/HEMV calls against their streaming kernels' time
(library event brackets) over a sequence of shapes in one process:
python scripts/sequence_probe.py dsymv:65536,zhemv:16384 ('clear' frees the
library caches between two calls)."""
import sys, json, torch
sys.path.insert(0, '/root/repo')
from bench import OPS, alg_bytes
from paper_1410_1726_b200 import _lib
from paper_1410_1726_b200.core import precision
lib=_lib.load()
st=torch.cuda.current_stream().cuda_stream
def run(opname, n):
    tag, fam, op, herm = OPS[opname]; p=precision(tag)
    name={("s",False):"ssymv",("d",False):"dsymv",("c",True):"chemv",("z",True):"zhemv"}[(tag,herm)]
    fn=getattr(lib, f"kblas_{name}_async")
    A=torch.empty(n,n,dtype=p.torch_dtype,device='cuda'); (torch.view_as_real(A) if p.is_complex else A).uniform_(-1,1)
    x=torch.ones(n,dtype=p.torch_dtype,device='cuda'); y=torch.empty_like(x)
    one,zero=_lib.scalar(tag,1.0),_lib.scalar(tag,0.0)
    call=lambda: fn(op.encode(), n, one, A.data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
    for _ in range(5): call()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): call()
    e1.record(); torch.cuda.synchronize()
    tot=e0.elapsed_time(e1)/10
    _lib.timing_read(); _lib.timing_enable(True)
    for _ in range(10): call()
    torch.cuda.synchronize(); _lib.timing_enable(False)
    ms,k=_lib.timing_read()
    b=alg_bytes(tag,'symv',n,n,op)
    print(json.dumps({"op":opname,"n":n,"call_gbs":round(b/(tot*1e-3)/1e9),"kernel_gbs":round(b/((ms/max(k,1))*1e-3)/1e9),"call_us":round(tot*1e3,1),"kernel_us":round(ms/max(k,1)*1e3,1)}), flush=True)
    del A; torch.cuda.empty_cache()
import os
seq = [tuple(x.split(":")) for x in (sys.argv[1] if len(sys.argv) > 1 else
       "dsymv:16384,dsymv:32768,dsymv:65536,zhemv:16384,zhemv:32768,zhemv:65536,ssymv:16384,ssymv:32768,ssymv:65536,ssymv:32768").split(",")]
for o, n in seq:
    if o == "clear":
        lib.kblas_clear_cache()
        continue
    run(o, int(n))
