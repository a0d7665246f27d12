"""Host simulation: how much a plan-time slot layout (per-line XOR keys, or full 4-channel chunk
permutations within each 128-byte line) could cut the RQ gather bank conflicts at K = 4096
(profiles/rq_r02.md: 3.17 -> 2.56 / 2.40 wavefronts per gather step; not implemented)."""
import numpy as np
rng=np.random.default_rng(1)
K=4096; n=(2240,1184,672)
perm=rng.permutation(K)
# steps: for each segment, chunk c (16 blocks), step q (0..15): lanes l -> position segoff+32*(16c+l//2)+16*(l%2)+q
steps=[]
off=0
for g in range(3):
    nb=(n[g]+127)//128*128//32  # padded blocks
    nch=(nb+15)//16
    for c in range(nch):
        for q in range(16):
            ch=[]
            for l in range(32):
                kb=16*c+l//2
                pos=32*kb+16*(l%2)+q
                if pos<n[g]: ch.append(perm[off+pos])
                else: ch.append(perm[off])  # pad lanes read block 0
            steps.append(np.array(ch))
    off+=n[g]
steps=np.array(steps)           # [S,32]
def bank(ch,key,mode):
    if mode=='xor_even': return 4*(((ch>>2)&7)^key[ch>>5])+(ch&3)
    if mode=='perm8': return 4*key[ch>>5][(ch>>2)&7]+(ch&3)
def cost(key,mode):
    b=bank(steps,key,mode)
    tot=0
    for r in range(len(b)):
        u=np.unique(steps[r]); bb=bank(u,key,mode)
        tot+=np.bincount(bb,minlength=32).max()
    return tot
base=cost(np.zeros(K//32,dtype=int),'xor_even')
print("steps",len(steps),"base wavefronts/step",base/len(steps))
key=np.zeros(K//32,dtype=int)
# which steps involve each line
line_steps=[set() for _ in range(K//32)]
for s,row in enumerate(steps):
    for ch in row: line_steps[ch>>5].add(s)
def step_cost(s,key):
    u=np.unique(steps[s])
    return np.bincount(bank(u,key,'xor_even'),minlength=32).max()
for it in range(3):
    improved=0
    for L in range(K//32):
        ss=list(line_steps[L])
        best=None
        for k in (0,2,4,6):
            old=key[L]; key[L]=k
            c=sum(step_cost(s,key) for s in ss)
            if best is None or c<best[0]: best=(c,k)
            key[L]=old
        if best[1]!=key[L]: improved+=1
        key[L]=best[1]
    print("iter",it,"wavefronts/step",cost(key,'xor_even')/len(steps),"changed",improved)

# full within-line chunk permutation (perm8): key[L] = permutation of 8 positions
pk=[list(range(8)) for _ in range(K//32)]
def bank8(u):
    return np.array([4*pk[c>>5][(c>>2)&7]+(c&3) for c in u])
def sc8(s):
    u=np.unique(steps[s]); return np.bincount(bank8(u),minlength=32).max()
tot=sum(sc8(s) for s in range(len(steps)))
print("perm8 base",tot/len(steps))
import itertools
for it in range(3):
    ch=0
    for L in range(K//32):
        ss=list(line_steps[L])
        cur=sum(sc8(s) for s in ss)
        for a,b in itertools.combinations(range(8),2):
            pk[L][a],pk[L][b]=pk[L][b],pk[L][a]
            c=sum(sc8(s) for s in ss)
            if c<cur: cur=c; ch+=1
            else: pk[L][a],pk[L][b]=pk[L][b],pk[L][a]
    print("perm8 iter",it,sum(sc8(s) for s in range(len(steps)))/len(steps),"changes",ch)
