import json,numpy as np
for f in ['/tmp/old.json','/tmp/new.json']:
    d=json.load(open(f))
    for k in ['cfg2','cfg5','cfg4','cfg3_tol']:
        a=np.load(d[k]['phi']); print(f,k,'nan',int(np.isnan(a).sum()),'inf',int(np.isinf(a).sum()))
