import numpy as np, torch, oracle, pfinputs
import paper_1202_6163_b200 as pf
dev=torch.device('cuda:0')
bad=0
for scheme in ('stratified','systematic'):
    for P in (2,3,7,16,1000,4097,8192,8193,20000,65536):
        for var in (0.1,1.0,10.0):
            x=pfinputs.gaussian_logw(P,var,seed=P*7+int(var*10))
            g=torch.from_numpy(x).to(dev)
            for seed in (1,2,3):
                a=getattr(pf,f'pf_resample_{scheme}')(g,seed).cpu().numpy()
                _,w=oracle.resample(scheme,x,seed)
                if not np.array_equal(a,w):
                    bad+=1
                    d=np.nonzero(a!=w)[0]
                    if bad<12: print(scheme,P,var,seed,'ndiff',len(d),d[:5],a[d[:5]],w[d[:5]])
print('bad',bad)
