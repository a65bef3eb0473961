import json, math, os, sys
sys.path.insert(0, '/root/repo')
from paper_1410_1726_b200 import tuner
from paper_1410_1726_b200.core import precision
V={'d':4,'s':8,'c':4,'z':2}
cfgs={0:(16,4,8),1:(8,4,8),2:(8,2,8),3:(8,4,16),4:(8,2,16),5:(4,4,16),6:(16,2,8),7:(8,8,8)}
rows=[('c',3548,5016,11),('c',7095,10033,17),('d',3548,5016,11),('d',7095,10033,17),('s',7095,10033,11),('s',33777,38858,17),('z',1774,2508,15)]
for tag,lo,hi,sh in rows:
    sizes=sorted({int(round(math.exp(math.log(lo)+f*(math.log(hi)-math.log(lo)))/32)*32) for f in [i/9 for i in range(10)]})
    pts=tuner.sweep('gemv', precision(tag), sizes, [tuner.auto_config('gemv'), tuner.TuneConfig(0,0)], reps=20, passes=2)
    NW,LR,U=cfgs[sh-10]; RB=LR*V[tag]
    out=[]
    for n in sizes:
        a=next(p for p in pts if p.size==n and p.config.is_auto).measured_gbs
        b=next(p for p in pts if p.size==n and not p.config.is_auto).measured_gbs
        P=math.ceil(n/RB)
        out.append(f"{n}:P{P}:{a/b:.2f}")
    print(tag, lo, hi, sh, ' '.join(out), flush=True)
