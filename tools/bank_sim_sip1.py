"""Shared-memory bank-conflict simulator for the line stages of k_sip_axis<1> (Q1 pressure):
wavefronts per warp-group of 8 cells for x-pitch PX, component pad, cell-stride pad and item order
(64-bit accesses: two half-warps, wavefronts = max distinct addresses per 8-byte bank slot).
The CF layout in fast_axis.cuh (PX 3, stride 122, cell-fastest) is the 80-wavefront optimum."""
import itertools
N=2; NF=4; NB=8; CPW=8
def wav(addrs):  # addrs: list of (lane, double index) active lanes; 64-bit: two half-warps
    tot=0
    for h in (0,1):
        banks={}
        for ln,a in addrs:
            if ln//16!=h: continue
            banks.setdefault(a%16,set()).add(a)
        tot+=max((len(v) for v in banks.values()),default=0)
    return tot
def sim(PX, CTpad, PERpad, order):
    PY=PX*N; CT=PY*N+CTpad
    O_U,O_SX,O_SY,O_SZ,O_UX=0,CT,2*CT,3*CT,4*CT
    PER=5*CT+61+PERpad
    idx=lambda i,j,k:i+PX*j+PY*k
    total=0; ideal=0
    def run(nitems, fn):
        nonlocal total, ideal
        for rnd in range((nitems+31)//32):
            insts={}
            for lane in range(32):
                it=lane+32*rnd
                if it>=nitems: continue
                for key,a in fn(it):
                    insts.setdefault(key,[]).append((lane,a))
            for key,ad in insts.items():
                total+=wav(ad); ideal+= (1 if all(l<16 for l,_ in ad) or all(l>=16 for l,_ in ad) else 2)
    def A(it):
        cl,r=divmod(it,12)
        if order=='cellfast':
            r,cl=divmod(it,CPW)
        d,tl=divmod(r,4); p,q=tl%2,tl//2
        st=[1,PX,PY][d]; b0=[idx(0,p,q),idx(p,0,q),idx(p,q,0)][d]
        base=cl*PER
        out=[]
        for l in range(N): out.append((('Ar',l),base+O_U+b0+l*st))
        for l in range(N): out.append((('Aw',l),base+[O_SX,O_SY,O_SZ][d]+b0+l*st))
        if d==0:
            for i in range(N): out.append((('Aux',i),base+O_UX+b0+i))
        return out
    run(CPW*12, A)
    def B(it):
        cl,tl=divmod(it,4)
        if order=='cellfast': tl,cl=divmod(it,CPW)
        b0=idx(0,tl%2,tl//2); base=cl*PER; o=[]
        for l in range(N): o+= [(('Bra',l),base+O_SY+b0+l),(('Brb',l),base+O_SZ+b0+l),(('Bwa',l),base+O_SY+b0+l),(('Bwb',l),base+O_SZ+b0+l)]
        return o
    run(CPW*4,B)
    def Cs(it):
        cl,tl=divmod(it,4)
        if order=='cellfast': tl,cl=divmod(it,CPW)
        b0=idx(tl%2,0,tl//2); base=cl*PER; o=[]
        for l in range(N):
            o+=[(('C1',l),base+O_UX+b0+l*PX),(('C2',l),base+O_SX+b0+l*PX),(('C3',l),base+O_SZ+b0+l*PX),(('C4',l),base+O_SY+b0+l*PX),
                (('C5',l),base+O_SX+b0+l*PX),(('C6',l),base+O_SZ+b0+l*PX)]
        return o
    run(CPW*4,Cs)
    def D(it):
        cl,tl=divmod(it,4)
        if order=='cellfast': tl,cl=divmod(it,CPW)
        b0=idx(tl%2,tl//2,0); base=cl*PER; o=[]
        for l in range(N):
            o+=[(('D1',l),base+O_SX+b0+l*PY),(('D2',l),base+O_SZ+b0+l*PY),(('D3',l),base+O_U+b0+l*PY)]
        return o
    run(CPW*4,D)
    return total, ideal, PER
print("current", sim(3,0,0,'cellmajor'))
res=[]
for PX in (2,3,4,5):
  for CTpad in range(0,8):
    for PERpad in range(0,16):
      for order in ('cellmajor','cellfast'):
        t,i,per=sim(PX,CTpad,PERpad,order); res.append((t,PX,CTpad,PERpad,order,per,i))
res.sort()
for r in res[:12]: print(r)
