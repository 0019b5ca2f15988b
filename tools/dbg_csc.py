import sys, time, faulthandler, numpy as np
faulthandler.dump_traceback_later(50, exit=True)
sys.path.insert(0, '.')
import torch, gen, paper_2209_07552_b200 as M
A = gen.Sparse(fmt="csr", m=4, n=4, ptr=np.array([0,2,3,3,5],np.int64), idx=np.array([0,2,1,0,3],np.int32), val=np.arange(1,6,dtype=np.float64))
T = gen.transpose(A)
ctx = M.Context(0,1,None,0,1)
print("partition...", flush=True); t=time.time()
ctx.partition("csc", 4, 4, ptr=T["ptr"], idx=T["idx"], val=T["val"])
print("partition ok %.2fs" % (time.time()-t), ctx.stats(), flush=True)
x = torch.ones(4, dtype=torch.float64, device="cuda"); y = torch.zeros(4, dtype=torch.float64, device="cuda")
ctx.spmv(1.0, x, 0.0, y); torch.cuda.synchronize(); print("spmv ok", y.cpu().numpy(), flush=True)
