"""Shared-memory bank-conflict model used to pick the v11 line kernel's X0 / X1
layout (row stride RS, plane stride PS) per lx: wavefronts of the row,
j-line and column access patterns of 32 lanes (8-B accesses)."""
import itertools
def wf(addrs):
    slots={}
    for a in set(addrs): slots.setdefault(a%16,set()).add(a)
    return max(len(v) for v in slots.values())
def cost(lx, RS, PS, ES, epc, pad=0):
    L2=lx*lx; nt=epc*L2
    tot={'A':0,'B':0,'C':0,'G':0,'H':0}
    for w in range(0,nt,32):
        lanes=range(w,min(w+32,nt))
        def dec(t):
            el=t//L2; r=t%L2; return el, r//lx, r%lx
        for c in range(lx):
            tot['A']+=wf([dec(t)[0]*ES+dec(t)[1]*PS+dec(t)[2]*RS+c+pad for t in lanes])
            tot['B']+=wf([dec(t)[0]*ES+dec(t)[1]*PS+c*RS+dec(t)[2]+pad for t in lanes])
            tot['C']+=wf([dec(t)[0]*ES+c*PS+dec(t)[1]*RS+dec(t)[2]+pad for t in lanes])
            tot['G']+=wf([dec(t)[0]*ES+0*PS+dec(t)[1]*RS+c+pad for t in lanes])
            tot['H']+=wf([dec(t)[0]*ES+0*PS+c*RS+dec(t)[2]+pad for t in lanes])
    return tot
import sys
for lx in range(5,17):
    L2=lx*lx
    best=None
    ideal=None
    for epc in ([1,2] if lx<=11 else [1]):
        nt=epc*L2
        lin=cost(lx,lx,L2,L2*lx,epc)
        lin1=cost(lx,lx,L2,L2*lx,epc,1)
        res=[]
        for RS in range(lx,lx+5):
            for PP in range(0,9):
                PS=lx*RS+PP
                ES=lx*PS
                for EP in range(0,9 if epc>1 else 1):
                    c=cost(lx,RS,PS,ES+EP,epc)
                    s=c['A']+c['B']+c['C']
                    res.append((s,c['G']+c['H'],RS,PP,EP,c))
        res.sort(key=lambda r:(r[0],r[1]))
        s,gh,RS,PP,EP,c=res[0]
        print(f"lx={lx} epc={epc} warps={(nt+31)//32} best RS={RS} PS=lx*RS+{PP} EP={EP} ABC={s} {c}  | u-linear pad0 {lin} pad1 {lin1}")
