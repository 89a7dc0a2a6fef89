import sys, os, numpy as np, torch, json
sys.path.insert(0, '/root/repo')
from paper_2011_03602_b200.runtime import lib
for (m,n,k,lo) in [(1024,1024,1024,0.0),(4096,4096,4096,0.0),(512,512,512,-1.0)]:
    g = torch.Generator().manual_seed(0)
    a = (torch.rand(m,k,generator=g)*(1-lo)+lo).cuda(); b=(torch.rand(k,n,generator=g)*(1-lo)+lo).cuda()
    c = torch.empty(m,n,device='cuda')
    lib().b2o_gemm_f32(a.data_ptr(), b.data_ptr(), c.data_ptr(), m,n,k,0); torch.cuda.synchronize()
    rows = slice(0, 256)
    ref = (a[rows].double() @ b.double()).cpu().numpy(); got = c[rows].double().cpu().numpy()
    print(json.dumps({"mode": os.environ.get("B2O_GEMM_SPLIT","0"), "shape":[m,n,k,lo], "normwise": float(np.linalg.norm(got-ref)/np.linalg.norm(ref)), "elem": float(np.max(np.abs(got-ref)/np.abs(ref)))}))
