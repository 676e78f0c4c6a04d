"""Shared-memory bank check of the generated register passes (host only):
for every JIT pass of the given configs, evaluate each register pass's lane ->
element map and report the worst per-half-warp bank multiplicity (1 = no
conflict).  python scripts/bankcheck.py c5 c3"""
import re, sys
from collections import Counter
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from hsf_inputs import make_config
from paper_2502_06959_b200 import Plan
def sw(e): return e + (e>>4) + (e>>8) + (e>>12)
def check(src, c64=True):
    res=[]
    lines=src.split('\n')
    for i,l in enumerate(lines):
        m=re.search(r'const u32 b = (.*);', l)
        if not m or 'gi' not in l: continue
        expr=m.group(1).replace('u','')
        offs=[]
        for l2 in lines[i+1:i+25]:
            mm=re.search(r'v\[\d+\] = (?:s|pb_)\[sb \+ (\d+)u\]', l2)
            if mm: offs.append(int(mm.group(1)))
        worst=0
        for o in offs[:16]:
            c0=Counter(); c1=Counter()
            for lane in range(32):
                gi=lane
                b=eval(expr)
                a=sw(b)+o
                bank=(2*a)%32 if c64 else (4*a)%32
                (c0 if lane<16 else c1)[bank]+=1
            worst=max(worst,max(c0.values()),max(c1.values()))
        res.append(worst)
    return res
for cfg in sys.argv[1:]:
    inst=make_config(cfg)
    P=Plan(inst.text, inst.n_low, inst.blocks, dtype=inst.dtype)
    for v in (0,1):
        for h in (0,1):
            for i in range(12):
                s=P.pass_source(h,i,v)
                if s is None: break
                print(cfg,'variant',v,'half',h,'pass',i,'rpass worst-way',check(s, inst.dtype=='c64'))
