import sys
def plan(L):
    e={2:0,3:0,5:0,7:0}
    for p in e:
        while L%p==0: L//=p; e[p]+=1
    R=[]
    while e[2]>=4: R.append(16); e[2]-=4
    if e[2]==3: R.append(8)
    if e[2]==2: R.append(4)
    if e[2]==1: R.append(2)
    R+=[5]*e[5]+[3]*e[3]+[7]*e[7]
    return R
def wavefronts(addrs16):  # addrs in 16B units
    groups={}
    for a in set(addrs16): groups.setdefault(a%8,set()).add(a)
    return max(len(s) for s in groups.values())
def pidx(e, pad): return e + (e>>pad) if pad else e
def stage_cost(Lt, C, R, L, pad, swz=None):
    Ls=L//R; nb=(Lt//R)*C; logC=C.bit_length()-1
    tot=0; ideal=0
    for w0 in range(0, nb, 32):
        lanes=range(w0, min(w0+32, nb))
        for r in range(R):
            ad=[]
            for q in lanes:
                c=q&(C-1); t=q>>logC; g=t//Ls; j=t%Ls
                e=((g*L+j)<<logC)+c + r*(Ls<<logC)
                ad.append(swz(e) if swz else pidx(e,pad))
            tot+=wavefronts(ad); ideal+=max(1,(len(ad)+7)//8)
    return tot, ideal
def report(Lt, C, pad, swz=None, label=''):
    R=plan(Lt); L=Lt; T=0; I=0; out=[]
    for r in R:
        t,i=stage_cost(Lt,C,r,L,pad,swz); T+=t; I+=i; out.append(f"R{r}:{t/i:.2f}"); L//=r
    print(f"{label} Lt={Lt} C={C} pad={pad} plan={R} total excess={T/I:.2f} ", ' '.join(out))
for Lt,C in [(1344,4),(4096,1),(280,8),(2240,1),(5000,2),(12000,1)]:
    for pad in (4,3,5):
        report(Lt,C,pad)
print("---- quarter-warp model")
def wavefronts(addrs16):
    tot=0
    for qtr in range(0,len(addrs16),8):
        groups={}
        for a in set(addrs16[qtr:qtr+8]): groups.setdefault(a%8,set()).add(a)
        tot+=max(len(s) for s in groups.values()) if groups else 0
    return tot
def stage_cost(Lt, C, R, L, pad, swz=None):
    Ls=L//R; nb=(Lt//R)*C; logC=C.bit_length()-1
    tot=0; ideal=0
    for w0 in range(0, nb, 32):
        lanes=range(w0, min(w0+32, nb))
        for r in range(R):
            ad=[]
            for q in lanes:
                c=q&(C-1); t=q>>logC; g=t//Ls; j=t%Ls
                e=((g*L+j)<<logC)+c + r*(Ls<<logC)
                ad.append(swz(e) if swz else pidx(e,pad))
            tot+=wavefronts(ad); ideal+=(len(ad)+7)//8
    return tot, ideal
for Lt,C in [(1344,4),(4096,1),(280,8),(2240,1),(5000,2),(12000,1)]:
    for pad in (4,3,5):
        report(Lt,C,pad)
    report(Lt,C,0,swz=lambda e: e ^ ((e>>3)&7), label='xor')
    report(Lt,C,0,swz=lambda e: e + (e>>3), label='pad8')
print("---- orderings")
def report2(Lt, C, R, pad, swz=None, label=''):
    L=Lt; T=0; I=0; out=[]
    for r in R:
        t,i=stage_cost(Lt,C,r,L,pad,swz); T+=t; I+=i; out.append(f"R{r}:{t/i:.2f}"); L//=r
    print(f"{label} Lt={Lt} C={C} pad={pad} plan={R} total excess={T/I:.2f} ", ' '.join(out))
def plan_odd_first(L):
    R=plan(L); odd=[r for r in R if r%2]; ev=[r for r in R if r%2==0]
    return sorted(odd,reverse=True)+sorted(ev)   # e.g. [7,5,3,...,2,4,8,16]
for Lt,C in [(1344,4),(2240,1),(5000,2),(12000,1),(280,8),(9600,1),(6250,2)]:
    for pad in (4,5,6):
        report2(Lt,C,plan_odd_first(Lt),pad,label='oddfirst')
