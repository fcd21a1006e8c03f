import itertools, random
def mmas_steady(BX):
    out=[]
    for j in range(BX+2):
        dhi=min(j,2); dlo=max(j-BX+1,0)
        out.append((j, j-dhi, j-dlo))   # slices [j-dhi, j-dlo]
    return out
def mmas_first(BX):
    out=[('z',x,x,x) for x in range(BX)]  # d=0 init, acc=0
    for j in range(1,BX+2):
        dhi=min(j,2); dlo=max(j-BX+1,1)
        out.append(('a',j,j-dhi,j-dlo))
    return out
def overl(a,b): return not (a[-1]<b[-2] or b[-1]<a[-2])
def score(seq, cyclic):
    n=len(seq); best=(99,0)
    # min gap between overlapping pairs (consecutive positions), count of gap-1 conflicts
    gaps=[]
    for i in range(n):
        for d in (1,2):
            if not cyclic and i+d>=n: continue
            if overl(seq[i], seq[(i+d)%n]): gaps.append(d)
    return (min(gaps) if gaps else 9, -gaps.count(1), -gaps.count(2))
def search(items, cyclic, fixed_prefix=None, iters=200000):
    best=None;bs=None
    for _ in range(iters):
        s=items[:]; random.shuffle(s)
        if fixed_prefix: 
            s=fixed_prefix+[x for x in s if x not in fixed_prefix]
        sc=score(s,cyclic)
        if bs is None or sc>bs: bs,best=sc,s
    return best,bs
random.seed(1)
for BX in (2,3,4,6,8):
    st,ss=search(mmas_steady(BX),True)
    print('steady',BX,[m[0] for m in st],ss)
    f=mmas_first(BX)
    # zero-init MMAs must precede any accumulate MMA on the same slice
    best=None;bs=None
    for _ in range(100000):
        s=f[:]; random.shuffle(s)
        ok=True; inited=set()
        for m in s:
            if m[0]=='z': inited.add(m[1])
            else:
                if any(x not in inited for x in range(m[2],m[3]+1)): ok=False;break
        if not ok: continue
        sc=score([m[1:] for m in s],False)
        if bs is None or sc>bs: bs,best=sc,s
    print('first',BX,[(m[0],m[1]) for m in best],bs)
