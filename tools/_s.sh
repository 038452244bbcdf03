python -m paper_2310_02065_b200.build >/dev/null
for shape in "3072 1040" "1024 1040" "4096 1040" "1024 4160"; do
  timeout 60 python tools/ablate.py $shape 16384 64 10 0 0 0 | grep -v host
done
timeout 120 python -c "
import torch,statistics
for (R,K) in [(3072,1024),(1024,1024),(4096,1024),(1024,4096)]:
    W=torch.randn(R,K,device='cuda').half(); X=torch.randn(16384,K,device='cuda').half()
    for _ in range(3): torch.matmul(X,W.t())
    torch.cuda.synchronize()
    ts=[]
    for _ in range(10):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); a.record(); torch.matmul(X,W.t()); b.record(); ts.append((a,b))
    torch.cuda.synchronize(); print('dense',R,K,statistics.median(a.elapsed_time(b) for a,b in ts)*1e3,'us')
"
