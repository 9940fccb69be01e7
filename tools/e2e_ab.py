import sys,time,os; sys.path.insert(0,".")
import numpy as np, torch
from paper_1303_1651_b200 import genmat
from paper_1303_1651_b200.kernels import multiply_rowmajor
from paper_1303_1651_b200.formats import CsrMatrix
a,b,_=genmat.config_operands(sys.argv[1])
def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype); out[...] = arr; return out
ap=CsrMatrix(a.rows,a.cols,pinned(a.row_ptr),pinned(a.col_idx),pinned(a.values))
bp=ap if b is a else CsrMatrix(b.rows,b.cols,pinned(b.row_ptr),pinned(b.col_idx),pinned(b.values))
w=[multiply_rowmajor(ap,bp) for _ in range(2)]; del w
ts=[]
for i in range(7):
    t=time.perf_counter(); c=multiply_rowmajor(ap,bp); ts.append((time.perf_counter()-t)*1e3)
print(sys.argv[1], os.environ.get("SPMMM_NO_NARROW"), os.environ.get("SPMMM_WIDEN_THREADS"), "median ms %.2f min %.2f" % (np.median(ts), min(ts)), flush=True)
