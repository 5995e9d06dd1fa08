import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, pa_synth as syn, paper_1805_02372_b200 as pa
def dw(w):
    w = np.ascontiguousarray(w).view(np.int32)
    return torch.from_numpy(np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])).cuda()
n,m,lim=20000,7000,5000
sw=syn.random_bits(syn.seed_stream(91+n), n+m-1); kw=syn.random_bits(syn.key_stream(91,n), n)
s=oracle.unpack(sw,n+m-1); x=oracle.unpack(kw,n)
mb=((lim//2)//32)*32; nb=lim+1-mb
st=dw(sw)
for r0 in (0,):
    r1=min(r0+mb,m)
    for c0 in range(0,n,nb):
        c1=min(c0+nb,n); ng=c1-c0; o=r0+n-c1
        want=oracle.toeplitz_bits(ng, r1-r0, s[o:o+ng+(r1-r0)-1], x[c0:c1])
        for route in ("bitpacked","transform"):
            h=pa.Hasher(ng, r1-r0, st, route=route, seed_bit_offset=o, allow_wide=True)
            got=oracle.unpack(h.hash(dw(oracle.pack(x[c0:c1]))).cpu().numpy().view(np.uint32), r1-r0)
            print(c0, ng, r1-r0, o, route, np.array_equal(got,want), flush=True)
            h.close()
out = torch.zeros(((m + 31) // 32 + 3,), dtype=torch.int32, device="cuda")
pa.pa_hash_blocked(n, m, st.data_ptr(), dw(kw).data_ptr(), out.data_ptr(), lim, 0)
torch.cuda.synchronize()
got=oracle.unpack(out.cpu().numpy().view(np.uint32), m); want=oracle.toeplitz_bits(n,m,s,x)
bad=np.flatnonzero(got!=want); print("blocked bad", bad.size, bad[:10], bad[-10:] if bad.size else None)
