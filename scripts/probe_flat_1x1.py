"""1x1 layers as one row of H*W pixels (r02b): FP32 SIMT time of Table-1 1x1 layers as given and flattened, AUTO and forced tiles."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_09808_b200 import conv
from paper_2101_09808_b200.inputs import Shape, make_inputs
from scripts.simt_sweep4 import timeit
cases = [((1,28269,1024,17,17), [None]), ((1,28269,1024,1,289), [None, "ver=2,tk=8,tw=8,kg=8,pw=2,bc=8", "ver=2,tk=8,tw=8,kg=4,pw=4,bc=8", "ver=2,tk=8,tw=8,kg=8,pw=1,bc=8", "ver=2,tk=4,tw=8,kg=8,pw=2,bc=8", "ver=2,tk=8,tw=4,kg=8,pw=2,bc=8"]),
         ((1,512,1024,17,17), [None]), ((1,512,1024,1,289), [None, "ver=2,tk=8,tw=8,kg=8,pw=2,bc=8,splits=8", "ver=2,tk=8,tw=4,kg=8,pw=2,bc=8,splits=8"]),
         ((1,256,512,34,34), [None]), ((1,256,512,1,1156), [None, "ver=2,tk=8,tw=8,kg=8,pw=2,bc=8,splits=4"]),
         ((1,64,128,136,136), [None]), ((1,64,128,1,18496), [None])]
for (N,K,C,H,W), specs in cases:
    sh = Shape(N=N,K=K,C=C,H=H,W=W,R=1,S=1)
    xi, wi = make_inputs(sh, seed=0)
    i, k = xi.cuda(), wi.cuda()
    for spec in specs:
        try:
            plan = conv.ConvPlan(*sh.as_tuple(), path="fp32_simt", tile=spec)
        except conv.ConvError as e:
            print(json.dumps({"shape": sh.as_tuple(), "spec": spec, "error": str(e)[:80]})); continue
        o, ws = plan.new_output(), plan.new_workspace()
        us = timeit(plan, i, k, o, ws)
        d = plan.describe()
        print(json.dumps({"shape": sh.as_tuple(), "spec": spec, "tile": d["tile"], "us": round(us, 1), "model_us": round(d["model"]["model_us"], 1)}), flush=True)
