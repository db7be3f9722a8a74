python - <<'PY'
import torch, paper_2205_09120_b200 as lb
M=N=8192; K=4096
fl=torch.empty(256<<20,dtype=torch.uint8,device='cuda')
a=lb.generate(1,45,0,M,K)
w=lb.prepare_weights(lb.pack_b(lb.encode_binary(lb.generate(1,45,1,K,N))))
c=torch.empty((M,N),dtype=torch.int16,device='cuda')
for lay in (2,0):
    ap=lb.encode_binary(a,layout=lay)
    for _ in range(3): lb.gemm_lowbit(0,ap,w,(M,N,K),kernel=2,out=c)
    ts=[]
    for _ in range(10):
        fl.zero_(); s,e=torch.cuda.Event(True),torch.cuda.Event(True); s.record(); lb.gemm_lowbit(0,ap,w,(M,N,K),kernel=2,out=c); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); print("c3 layout",lay,f"{ts[5]:.4f} ms {2*M*N*K/ts[5]/1e9:.0f} TOPS")
PY
