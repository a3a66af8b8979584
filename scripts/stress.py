"""Back-to-back launch stress test (hang / race detection), GPU box."""
import sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_10876_b200 as tw
li = int(sys.argv[1]) if len(sys.argv) > 1 else 0
use_graph = len(sys.argv) > 2 and sys.argv[2] == "graph"
LAYERS = [(768, 768), (768, 3072), (3072, 768)]
k, n = LAYERS[li]
w = tw.round_to(tw.synthetic_matrix(0, k, n, 0), "fp16")
_, tsm = tw.prune_tw(w, 0.75, 128)
plan = tw.TwPlan(tw.encode_cto(tsm))
a = tw.round_to(tw.synthetic_matrix(0, 8192, k, 1), "fp16")
at = plan.prepare(torch.from_numpy(a).cuda())
out = torch.empty((tsm.n_condensed, 8192), dtype=torch.float16, device="cuda")
ref = plan.run(at).float()
torch.cuda.synchronize()
for it in range(1, 65):
    t0 = time.time()
    if use_graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(it):
                    plan.run(at, out=out)
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
    else:
        for _ in range(it):
            plan.run(at, out=out)
    torch.cuda.synchronize()
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"layer {li} graph={use_graph} launches {it}: ok err {err:.2e} {time.time()-t0:.3f}s", flush=True)
