import numpy as np, torch, oracle, pfinputs
import paper_1202_6163_b200 as pf
dev=torch.device('cuda:0')
rng=np.random.default_rng(2)
bad=0
for P in (1,3,8,4096,8191,8193,30000,65536):
    for scheme,var in (("systematic",10.0),("multinomial",1.0),("stratified",0.1)):
        x=pfinputs.gaussian_logw(P,var,seed=P+1)
        _,anc=oracle.resample(scheme,x,17)
        if scheme=="multinomial": anc=rng.permutation(anc).astype(np.int32)
        perm=pf.pf_permute(torch.from_numpy(anc).to(dev)).cpu().numpy()
        w=oracle.permute(anc)
        if not np.array_equal(perm,w):
            bad+=1; d=np.nonzero(perm!=w)[0]
            print(P,scheme,'ndiff',len(d),d[:6],perm[d[:6]],w[d[:6]], 'o-sum', np.bincount(anc,minlength=P).sum())
print('bad',bad)
