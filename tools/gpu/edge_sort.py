import numpy as np, torch, sys, time
sys.path.insert(0,'.')
import paper_1712_04732_b200 as se
# a coincident-z layer: every particle of a column in one fine bin
rng=np.random.default_rng(1)
N=40000; L=4.0
pos=rng.random((N,3))*L; pos[:,2]=1.2345
q=rng.uniform(-1,1,N); q-=q.mean()
s=se.ParticleSystem(pos,q,L)
p=se.SEParams(xi=6.0,rc=0.5,M=32,P=8,window="bm",shape=20.0)
t=time.time(); a=se.real_space_sum(s,6.0,0.5,se.Periodicity(3)); print("layer real space", time.time()-t)
se.set_deterministic(True)
b1=se.total_potential(s,p,se.Periodicity(3)); b2=se.total_potential(s,p,se.Periodicity(3))
print("det layer bitwise", np.array_equal(b1,b2))
se.set_deterministic(False)
c=se.total_potential(s,p,se.Periodicity(3)); print("det vs default", se.relative_rms_error(b1,c))
# tiny systems
for n in (1,2,3):
    pp=rng.random((n,3)); qq=np.zeros(n) if n==1 else rng.uniform(-1,1,n); qq-=qq.mean()
    print(n, se.total_potential(se.ParticleSystem(pp,qq,1.0), se.SEParams(xi=6.0,rc=0.4,M=16,P=4,window="bm",shape=10.0), se.Periodicity(3)))
