import sys, os, torch, statistics
sys.path.insert(0, os.getcwd())
from paper_2511_13061_b200 import macko as M
R,C=36864,12288
dense=torch.empty((R,C),dtype=torch.float16,device="cuda"); M.gen_dense(dense,R,C,0.5,seed=1234)
dm=M.DeviceMatrix.from_dense(dense); del dense
x=torch.empty(C,dtype=torch.float16,device="cuda"); M.gen_vector(x,C,seed=4321)
y=torch.empty(R,dtype=torch.float16,device="cuda")
st=torch.cuda.current_stream()
flush=torch.ones(256<<20,dtype=torch.float32,device="cuda")
for mode in [-1]:
  ts=[]
  for i in range(60):
    flush.sum()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record(st); dm.spmv_into(x,y,st); b.record(st); b.synchronize(); ts.append(a.elapsed_time(b)*1e3)
  print(mode, [round(t,1) for t in ts])
  print("median", statistics.median(ts), "mean", sum(ts)/len(ts))
