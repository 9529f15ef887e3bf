#!/usr/bin/env bash
O=gpurun_out/r2u
mkdir -p $O
timeout 600 python -m pytest tests/test_mha_gpu.py tests/test_random_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -3 | tee $O/pytest.log
# bitwise: speculative vs non-speculative forward on random inputs with large score growth
cat > /tmp/bw.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2502_12784_b200 as vb
out = {}
for (B,H,N,d,causal,dt) in [(2,4,2048,128,1,torch.bfloat16),(1,2,1000,64,0,torch.float16),(1,2,3000,128,0,torch.float16)]:
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    q,k,v = (torch.randn(B,H,N,d,generator=g,device="cuda")*(4.0 if i==0 else 1.0) for i in range(3))
    # scores that grow along the keys: forces lazy rescales mid-row
    k = k * torch.linspace(0.2, 3.0, N, device="cuda").view(1,1,N,1)
    q,k,v = (x.to(dt) for x in (q,k,v))
    o, lse = vb.mha_forward(q,k,v,bool(causal))
    out[(B,H,N,d,causal)] = (o.cpu(), lse.cpu())
torch.save(out, sys.argv[1])
PY
python /tmp/bw.py $O/spec.pt && VATTN_LIB=tools/variants/nospec.so python /tmp/bw.py $O/nospec.pt && python -c "
import torch; a=torch.load('$O/spec.pt'); b=torch.load('$O/nospec.pt')
print('bitwise', all(torch.equal(a[k][0],b[k][0]) and torch.equal(a[k][1],b[k][1]) for k in a))"
timeout 600 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 nospec 2>&1 | tee $O/variants.txt
