import itertools, sys
sys.path.insert(0, '.')
from median27 import batcher
cells = [(p,q,r) for p in range(3) for q in range(3) for r in range(3)]
def ok(t):
    for p,q,r in cells:
        if p<2 and t[(p,q,r)]>t[(p+1,q,r)]: return False
        if q<2 and t[(p,q,r)]>t[(p,q+1,r)]: return False
        if r<2 and t[(p,q,r)]>t[(p,q,r+1)]: return False
    return True
pats=[]
for bits in itertools.product((0,1),repeat=27):
    pass
