python - <<'PY'
import torch, paper_2205_09120_b200 as lb
M,N,K=1048576,1024,2048
a=lb.generate(0,47,0,M,K); ap=lb.encode_ternary(a); del a
w=lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0,47,1,K,N))))
c=torch.empty((M,N),dtype=torch.int16,device='cuda'); fl=torch.empty(256<<20,dtype=torch.uint8,device='cuda')
for kern in (2,4):
    for _ in range(3): lb.gemm_lowbit(1,ap,w,(M,N,K),kernel=kern,out=c)
    ts=[]
    for _ in range(10):
        fl.zero_(); s,e=torch.cuda.Event(True),torch.cuda.Event(True); s.record(); lb.gemm_lowbit(1,ap,w,(M,N,K),kernel=kern,out=c); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); t=ts[5]; print("reference-layout planes kernel", kern, f"{t:.4f} ms {2*M*N*K/t/1e9:.0f} TOPS")
PY
