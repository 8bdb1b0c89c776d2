import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, golden_cases as G
from oracle import cgh_oracle as O
from paper_2006_10509_b200 import algorithms as A
from paper_2006_10509_b200.runtime import precision
rec=G.manifest()['cases']['gs_backprop_fresnel_32_pl16']
for variant in ['asis','random','fourier']:
    cfg,t,il=G.build(rec)
    if variant=='random': cfg.init_mode='random-phase'
    if variant=='fourier': cfg.propagation=type(cfg.propagation)()
    for k in (1,2,12):
        cfg.iterations=k
        _,r=O.gs(cfg,t,il,keep_fields=(k,))
        with precision('fp64'):
            idx,fld,rep,tr=A.gs_field(cfg,t,il)
        d=np.abs(fld-r.fields[k]); bad=np.argwhere(d>1e-9)
        print(variant,k,'maxdiff',d.max(),'nbad',len(bad), bad[:5].tolist(), 'trace', max(abs(a[1]-b[1]) for a,b in zip(tr,r.error_trace)))
