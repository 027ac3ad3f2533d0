"""Shared-memory bank-conflict simulator for fft_core.cuh's cta_fft access
patterns (float2 = 8 B words, a 64-bit warp access served per half-warp).
Prints, per N, the wavefronts of the current row / column strides
(fft::CtaLaunch) against the best stride in [SMEM, SMEM + 32]."""
import math
def plan(N):
    E = 32 if N>=32 else N; T=N//E; LOGN=int(math.log2(N)); LOGE=int(math.log2(E))
    P = 1 + (LOGN - LOGE + LOGE - 1)//LOGE
    radix=lambda p: E if p<P-1 else N//E**(P-1)
    return E,T,P,radix
def pad32(i): return i + (i>>5)
def wavefronts(addrs):  # addrs: list of float2 indices for 32 lanes (None = inactive)
    tot=0
    for h in (addrs[:16],addrs[16:]):
        banks={}
        for a in h:
            if a is None: continue
            for w in (2*a,2*a+1):
                banks.setdefault(w%32,set()).add(w)
        tot += max((len(s) for s in banks.values()), default=0)
    return tot
def accesses(N, lane_map, S):
    """lane_map(lane)->(slot, t) ; yields per-instruction address lists"""
    E,T,P,radix=plan(N); out=[]
    if P==1: return out
    lanes=[lane_map(l) for l in range(32)]
    for r in range(E):  # pass0 store
        out.append([s*S+pad32(t*E+r) for s,t in lanes])
    for p in range(1,P):
        R=radix(p); NS=E**p; Q=E//R
        for q in range(Q):
            for r in range(R):
                out.append([s*S+pad32(t+q*T + r*(N//R)) for s,t in lanes])
        if p<P-1:
            for q in range(Q):
                for r in range(R):
                    ad=[]
                    for s,t in lanes:
                        b=t+q*T; base=(b//NS)*NS*R+(b&(NS-1)); ad.append(s*S+pad32(base+r*NS))
                    out.append(ad)
    return out
def cost(N, lane_map, S):
    acc=accesses(N,lane_map,S)
    return sum(wavefronts(a) for a in acc), 2*len(acc)
def col_stride(smem, pc):
    if pc >= 16: return smem | 1
    if pc <= 1: return smem
    s = smem
    while s % (32 // pc) != 16 // pc: s += 1
    return s
for N in [64,128,256,512,1024,2048,4096,8192,16384]:
    E,T,P,radix=plan(N)
    PC = max(1, 256//T)
    smem=N+N//32
    cols_map=lambda l,warp=0: (l%PC, (warp*32+l)//PC)
    rows_map=lambda l: ((l//T) if T<32 else 0, l%T if T<32 else l)
    res=[]
    best=None
    for S in range(smem, smem+33):
        c,ideal=cost(N,cols_map,S); r,_=cost(N,rows_map,S)
        res.append((S,c,r,ideal))
    cur=col_stride(smem,PC)
    d={S:(c,r,i) for S,c,r,i in res}
    bc=min(res,key=lambda x:(x[1],x[0])); br=min(res,key=lambda x:(x[2],x[0]))
    print(N,'PC',PC,'col S',cur,'cols',d[cur][0],'rows(S=SMEM)',d[smem][1],'| best cols S',bc[0],bc[1],'best rows S',br[0],br[2])
