import os, sys, ctypes as C
os.environ["SBS_CEM_CLOCKS"]="1"
sys.path.insert(0,'.')
import numpy as np
from paper_2403_11383_b200 import binding as B, workloads as W
L=B.load_library(); L.sbs_debug_cem_clocks.argtypes=[C.c_void_p, C.POINTER(C.c_longlong)]
cfg,inputs=W.config3("cem")
c=B.Controller(cfg); c.set_reference(0, inputs[0]["xref"])
for it in range(5):
    c.step(inputs)
    t=(C.c_longlong*6)(); L.sbs_debug_cem_clocks(c.ctx, t)
    t=list(t); print([t[i+1]-t[i] for i in range(5)], 'total', t[5]-t[0])
