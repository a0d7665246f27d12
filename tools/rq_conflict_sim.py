"""Host simulation: shared-memory wavefronts of the RQ gather for random 512-channel chunks,
and how many a per-lane rotation of the gather order (multiples of 4) removes (profiles/rq_r02.md)."""
import numpy as np, itertools
rng=np.random.default_rng(0)
def wavefronts(chans, R):
    # chans: 32 channel ids read in one step; returns #wavefronts (max distinct words per bank)
    if R==1: words=chans>>1
    elif R==2: words=chans
    else: words=chans*2
    banks=words&31 if R<=2 else (words&31)
    d={}
    for w,b in zip(words,banks): d.setdefault(b,set()).add(w)
    return max(len(s) for s in d.values())
def chunk_cost(P, rot, R):
    # P: [32 lanes][16] channels; rot: per-lane rotation
    tot=0
    for q in range(16):
        ch=np.array([P[l][(q+rot[l])%16] for l in range(32)])
        tot+=wavefronts(ch,R)
    return tot
K=28672
for R in (1,2):
    base=[];opt=[]
    for trial in range(30):
        P=rng.permutation(K)[:512].reshape(32,16)
        rot=[0]*32
        c0=chunk_cost(P,rot,R); base.append(c0)
        # local search over rotations in {0,4,8,12}
        best=c0; improved=True
        while improved:
            improved=False
            for l in range(32):
                for r in (0,4,8,12):
                    if r==rot[l]: continue
                    old=rot[l]; rot[l]=r
                    c=chunk_cost(P,rot,R)
                    if c<best: best=c; improved=True
                    else: rot[l]=old
        opt.append(best)
    print(f"R={R}: wavefronts per chunk (16 steps): base {np.mean(base):.1f} ({np.mean(base)/16:.2f}/step)  rot4 {np.mean(opt):.1f} ({np.mean(opt)/16:.2f}/step)")
