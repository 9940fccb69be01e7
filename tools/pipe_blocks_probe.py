import sys,time; sys.path.insert(0,".")
import numpy as np, torch
from paper_1303_1651_b200 import genmat, _lib
from paper_1303_1651_b200.formats import CsrMatrix
def pinned(arr):
    buf = torch.empty(max(arr.nbytes, 1), dtype=torch.uint8, pin_memory=True)
    out = buf.numpy()[:arr.nbytes].view(arr.dtype); out[...] = arr; return out
for cfg in sys.argv[1:]:
    a,b,_=genmat.config_operands(cfg)
    ap=CsrMatrix(a.rows,a.cols,pinned(a.row_ptr),pinned(a.col_idx),pinned(a.values))
    bp=ap if b is a else CsrMatrix(b.rows,b.cols,pinned(b.row_ptr),pinned(b.col_idx),pinned(b.values))
    ctx=_lib.default_context()
    va=_lib.csr_view(ap.rows,ap.cols,ap.row_ptr,ap.col_idx,ap.values)
    vb=va if b is a else _lib.csr_view(bp.rows,bp.cols,bp.row_ptr,bp.col_idx,bp.values)
    for G in (4,8,12,16):
        w=[_lib.multiply_host(ctx,va,vb,6,0,G) for _ in range(2)]; del w
        ts=[]
        for i in range(5):
            t=time.perf_counter(); r=_lib.multiply_host(ctx,va,vb,6,0,G); ts.append((time.perf_counter()-t)*1e3); del r
        print(cfg, G, "median %.2f" % np.median(ts), flush=True)
