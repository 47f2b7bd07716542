import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2406_16499_b200 as P
from paper_2406_16499_b200 import generate as G
from oracle.oracle import Oracle
o=Oracle("ref")
for (m,n,p),k in [((200,100,50),1e3),((60,40,10),1e6),((120,80,30),1e7),((200,100,50),1e9),((1024,512,128),1e6)]:
    A,B,b,d=G.lse_problem(m,n,p,k,1e2,21+m+n)
    for pc in ("bd_split","left"):
        g=P.gmres_refine_lse(P.LseProblem(A,B,b,d),P.RefinementConfig(maxit=20),precond=pc)
        r=o.gmres_lse(A,B,b,d,maxit=20,precond=pc)
        fe=np.linalg.norm(g.state.x-r.x)/np.linalg.norm(r.x)
        print((m,n,p),k,pc,'gpu',g.trace.status,g.trace.iterations,g.trace.inner_iterations,'ref',r.status,r.iterations,r.inner,'fwd %.2e'%fe, 'phases', {kk:round(v,4) for kk,v in g.trace.timing.items()})
