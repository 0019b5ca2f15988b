"""CPU estimate: would sorting every split row's entries by (degree-ordered) compact x id make the slab
gathers coalesce?  R-MAT scale 24; counts, per group of 32 consecutive slab entries (one gather
instruction), the distinct 128-B lines of x' the cold entries touch (hot ids < 4096 excluded), in the
row's column order and sorted by compact id.  Result (profiles/r2_kernel_ab.txt #15): 103.0M -> 94.4M
line requests for 104.7M cold slab gathers -- only 8 % (4 % of all gathers): not built.
    PYTHONPATH=. python tools/slab_order_sim.py"""
import numpy as np, gen, time
t=time.time()
A=gen.make_config("rmat")
print("gen", time.time()-t, A.nnz, flush=True)
m=A["m"]; ptr=A["ptr"]; idx=A["idx"]
deg=np.bincount(idx, minlength=A["n"])
used=np.nonzero(deg)[0]
order=used[np.lexsort((used, -deg[used]))]     # degree desc, column asc
cmap=np.full(A["n"], -1, np.int64); cmap[order]=np.arange(order.size)
nhot=4096
lens=np.diff(ptr)
split=np.nonzero(lens>512)[0]
print("split rows", split.size, "slab nnz", lens[split].sum(), flush=True)
tot_cold=0; req_sorted=0; req_orig=0
for r in split:
    c=cmap[idx[ptr[r]:ptr[r+1]]]
    for arr,name in ((np.sort(c),'s'),(c,'o')):
        n=arr.size; g=(n+31)//32
        pad=np.full(g*32, -1, np.int64); pad[:n]=arr
        pad=pad.reshape(g,32)
        cold=(pad>=nhot)
        lines=np.where(cold, pad//16, -1)
        # distinct lines per group (excluding -1)
        s=np.sort(lines,axis=1)
        d=(np.diff(s,axis=1)!=0)&(s[:,1:]>=0)
        cnt=d.sum(1)+(s[:,0]>=0)
        if name=='s': req_sorted+=cnt.sum(); tot_cold+=cold.sum()
        else: req_orig+=cnt.sum()
print("slab cold gathers", tot_cold, "requests orig(lines)", req_orig, "sorted", req_sorted)
