import sys, json, torch
sys.path.insert(0, '/root/repo')
from bench import OPS, alg_bytes
from paper_1410_1726_b200 import _lib
from paper_1410_1726_b200.core import precision
lib=_lib.load()
st=torch.cuda.current_stream().cuda_stream
def t(opname, n, mid):
    prev=lib.kblas_set_symv_mid(mid)
    tag, fam, op, herm = OPS[opname]; p=precision(tag)
    name={("s",False):"ssymv",("d",False):"dsymv",("c",True):"chemv",("z",True):"zhemv"}[(tag,herm)]
    fn=getattr(lib, f"kblas_{name}_async")
    nc=max(1,min(8,-(-(1<<30)//(n*n*p.element_bytes))))
    As=[torch.empty(n,n,dtype=p.torch_dtype,device='cuda') for _ in range(nc)]
    for A in As: (torch.view_as_real(A) if p.is_complex else A).uniform_(-1,1)
    x=torch.ones(n,dtype=p.torch_dtype,device='cuda'); y=torch.empty_like(x)
    one,zero=_lib.scalar(tag,1.0),_lib.scalar(tag,0.0)
    call=lambda i: fn(op.encode(), n, one, As[i%nc].data_ptr(), n, x.data_ptr(), 1, zero, y.data_ptr(), 1, st)
    for i in range(6): call(i)
    torch.cuda.synchronize(); best=1e9
    for _ in range(3):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20): call(i)
        e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1)/20)
    plan=_lib.last_plan()
    lib.kblas_set_symv_mid(prev)
    del As; torch.cuda.empty_cache()
    return round(alg_bytes(tag,'symv',n,n,op)/(best*1e-3)/1e9), plan.split()[6] if len(plan.split())>6 else plan
for opname in ("ssymv","dsymv","chemv","ssymv_u"):
    for n in (12288,14336,16384,18432,20480):
        a=t(opname,n,12288); b=t(opname,n,1<<30)
        print(json.dumps({"op":opname,"n":n,"wide":a,"mid":b,"mid/wide":round(b[0]/a[0],3)}), flush=True)
