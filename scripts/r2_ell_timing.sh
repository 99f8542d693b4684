#!/bin/bash
# per-CTA section times of the panel mat-vec (library built with -DREGOT_PANEL_TIMING): last two launches of a short solve
mkdir -p gpurun_out
REGOT_B200_PANEL_AHEAD=7777 MAXIT=${MAXIT:-40} timeout 600 python scripts/solve_cloud.py D 0 > gpurun_out/r2_ell_timing.log 2>&1
grep "^panel cta" gpurun_out/r2_ell_timing.log | tail -296 > gpurun_out/r2_ell_timing_last.txt
python - <<'PY'
import re
rows=[l.split() for l in open('gpurun_out/r2_ell_timing_last.txt')]
def col(name): 
    return [int(r[r.index(name)+1]) for r in rows]
for half,(lo,hi) in (("first of the last two launches",(0,148)),("last launch",(148,296))):
    R=rows[lo:hi]
    if not R: continue
    g=lambda name:[int(r[r.index(name)+1]) for r in R]
    st=g("stage"); f=g("first"); m=g("mean"); l=g("last"); p23=g("pass23")
    dw=[int(r[r.index("defer")+1]) for r in R]; dc=[int(r[r.index("defer")+2]) for r in R]
    tot=[a+b+c for a,b,c in zip(st,l,p23)]
    mx=lambda v:(min(v),sum(v)//len(v),max(v))
    print(half,"stage",mx(st),"pass1 first-warp-done",mx(f),"mean",mx(m),"last",mx(l),"pass23",mx(p23),"total",mx(tot),"defer_w",mx(dw),"defer_c",mx(dc))
PY
