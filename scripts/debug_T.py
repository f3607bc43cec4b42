import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
import paper_2209_00315_b200 as pb
from oracle.ops import Discretisation
from synthetic import make_problem, random_state, initial_state
p = make_problem('T1'); d = Discretisation(p.verts,p.tris,p.K,p.rho_in,p.rho_f)
for st in ['init','rand','rand_phi0']:
    if st=='init': phi,rho,s = initial_state(p,1.0); mu=1.0
    else: phi,rho,s = random_state(p, seed=3, mu=1e-2); mu=1e-2
    if st=='rand_phi0': phi=np.zeros_like(phi)
    ctx = pb.Context(p.verts,p.tris,p.K,p.rho_in,p.rho_f)
    ctx.set_state(phi,rho,s,mu); ctx.assemble()
    rp,ci,cv = ctx.get_T()
    Tg = sp.csr_matrix((cv,ci,rp),shape=(d.m,d.m)).toarray()
    To = d.T_matrix(phi,rho,s).toarray()
    D = abs(Tg-To)
    r,c = np.unravel_index(D.argmax(), D.shape)
    print(st, 'maxdiff', D.max(), 'at', r, c, 'gpu', Tg[r,c], 'orc', To[r,c], 'nnz g/o', (Tg!=0).sum(), (To!=0).sum())
    print('  row', r, 'gpu cols', np.nonzero(Tg[r])[0][:40], '\n  orc cols', np.nonzero(To[r])[0][:40])
    print('  gpu vals', Tg[r][np.nonzero(Tg[r])[0]][:12], '\n  orc vals', To[r][np.nonzero(To[r])[0]][:12])
