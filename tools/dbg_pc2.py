import sys; sys.path.insert(0,".")
import numpy as np, synth, oracle
from paper_1709_01126_b200 import Pot3d
for dims in [(2,2,2),(3,5,7),(4,9,33),(5,17,70)]:
    rf,tf,pf=synth.grid(*dims)
    try:
        with Pot3d(rf,tf,pf,synth.br0_map(tf,pf,0),pc=2) as s:
            r=synth.random_vector(int(np.prod(dims)),3).reshape(dims[::-1])
            z=s.precond(r); zr=oracle.precond(rf,tf,pf,r,pc=2)
            print(dims, s.info()["pc"], np.abs(z-zr).max()/np.abs(zr).max(), flush=True)
    except Exception as e:
        print(dims, "ERR", e, flush=True)
