import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2605_30267_b200 import ot
from oracle import oracle as O
for (n,m) in [(5,5),(2,2),(37,23),(3,3000),(300,257)]:
    p=ot.synthetic_rescaled(n,m,33,0.6)
    v=np.linspace(-1,1,m); v-=v.mean()
    e=ot.eval_normalized_step(p,v)
    print(n,m,'f_gpu',e.f_value,'f_from_u',1-e.u.dot(p.a)-v.dot(p.b), 'oracle', O.eval_normalized_step(O.synthetic_rescaled(n,m,33,0.6),v)['f_value'])
