import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2407_12208_b200 as mpk, synth, oracle
for (n,d,k,dist) in [(1000,64,256,'fp16'),(4099,128,1024,'fp16'),(3001,32,64,'e5m2')]:
    X,_ = synth.blobs(n,d,10,seed=0,dtype=np.float32)
    Xn,_,_ = oracle.normalize(X,'zscore',work='fp32'); Xn=Xn.astype(np.float32)
    C = synth.init_rows(Xn,k,0)
    km = mpk.KMeans(n,d,k,'fp32',dist)
    mpk.kmeans_set_centroids(km.h, torch.from_numpy(C).cuda())
    lab = torch.empty(n,dtype=torch.int32,device='cuda')
    sse = km.assign(torch.from_numpy(Xn).cuda(), lab)
    torch.cuda.synchronize()
    ref,dmin,_ = oracle.assign(Xn,C,work='fp32',dist=dist)
    l = lab.cpu().numpy()
    print(n,d,k,dist,'match', (l==ref).mean(), 'sse', sse, np.maximum(dmin,0).sum(), flush=True)
    km.close()
