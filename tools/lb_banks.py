"""Shared-memory bank check for csrc/fwht_cols_lb.cu (the large-block left
transform): for every strip geometry, the round-1 staging reads, the
exchange writes / reads and the code-staging writes must need no more
wavefronts than their byte count does (0 = bank-optimal).
  python tools/lb_banks.py"""
from collections import defaultdict
def wf(acc):
    bw=defaultdict(set); tot=0
    for a,n in acc:
        for w in range(a//4,(a+n)//4): bw[w%32].add(w); tot+=4
    return max(len(s) for s in bw.values()), (tot+127)//128
def cfg(LB,E):
    B=1<<LB; W=E//B; NCP=W//2; NT=E//128; R2B=LB-6; R2=1<<R2B; C2=64//R2; NQ=NCP//C2; RB=4*W
    INL={16:3,32:2,64:1}.get(RB,0)
    return B,W,NCP,NT,R2,C2,NQ,RB,INL
def swz(r,cp,RB,INL):
    # lb_swz in fwht_cols_lb.cu
    o=r*RB+8*cp; f=(((r>>6)<<(0 if RB==16 else 1))^(r>>INL))&7; return o^(f<<4)
def run(LB,E,es):
    B,W,NCP,NT,R2,C2,NQ,RB,INL=cfg(LB,E)
    seen=set(swz(r,cp,RB,INL) for r in range(B) for cp in range(NCP)); assert len(seen)==B*NCP and max(seen)<B*RB
    bad=defaultdict(int)
    BOXS=65*W*es
    for w in range(NT//32):
        for j in range(64):
            a1=[];a2=[]
            for l in range(32):
                t=32*w+l; cp=t%NCP; g=t//NCP
                a1.append((g*BOXS+j*W*es+cp*2*es, 2*es))   # staging read
                a2.append((swz(64*g+j,cp,RB,INL),8))      # exchange write
            x,m=wf(a1); bad['stg']=max(bad['stg'],x-m)
            x,m=wf(a2); bad['xw']=max(bad['xw'],x-m)
        for i in range(R2):
            for c in range(0,C2,2 if C2>1 else 1):
                a=[]
                for l in range(32):
                    t=32*w+l; q=t%NQ; jp=t//NQ; cp=q*C2+c
                    o=swz(64*i+jp,cp,RB,INL)
                    if C2>1: assert swz(64*i+jp,cp+1,RB,INL)==o+8
                    a.append((o,16 if C2>1 else 8))
                x,m=wf(a); bad['xr']=max(bad['xr'],x-m)
        # code staging write (dense bytes r*W + 2*cp), per row i
        for i in range(0,R2, 2 if C2==1 else 1):
            a=[]
            for l in range(32):
                t=32*w+l; q=t%NQ; jp=t//NQ
                r=64*i+jp; nb=2 if C2==1 else 2*C2
                a.append((r*W+2*q*C2, nb if nb>=4 else 2))
            # sub-word stores: treat 2B as within word
            x,m=wf([(aa - aa%4, 4) if n<4 else (aa,n) for aa,n in a]); bad['cw']=max(bad['cw'],x-m)
    return dict(bad), (B,W,NCP,NT,R2,C2,NQ)

if __name__ == "__main__":
    worst = 0
    for es, LB, E in ((2, 9, 16384), (2, 10, 32768), (2, 11, 32768), (2, 12, 32768),
                      (4, 9, 16384), (4, 10, 16384), (4, 11, 16384), (4, 12, 16384)):
        bad, geo = run(LB, E, es)
        worst = max(worst, max(bad.values()))
        print("bf16" if es == 2 else "fp32", "B=%d" % (1 << LB), "E=%d" % E, bad, geo)
    raise SystemExit(1 if worst else 0)
