"""Stepper timing without instrumentation: refactor + tcg_step(n_t) with the library's CUDA
events (set_profile 7); prints ms per step and us per PCG iteration (incl. step overhead).
env: TORCH_STREAM=1 (solver on a torch stream), FLUSH=1 (256 MiB L2 flush before each pass)"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, workloads, paper_2510_23446_b200 as tcg
tag = os.environ.get("TAG", "")
use_torch = os.environ.get("TORCH_STREAM") == "1" or os.environ.get("FLUSH") == "1"
if use_torch:
    import torch
    stream = torch.cuda.Stream()
    flush = None if os.environ.get("LATE_FLUSH") == "1" else torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for name in sys.argv[1:] or ["cfg2"]:
    pr = workloads.get(name)
    s = (tcg.Solver(stream=stream.cuda_stream) if os.environ.get("TORCH_STREAM") == "1" else tcg.Solver()).configure(pr)
    s.setup()
    if use_torch and flush is None:
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    res = []
    for rep in range(int(os.environ.get('REPS', '3'))):
        if os.environ.get("FLUSH") == "1":
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
            torch.cuda.synchronize()
        s.refactor()
        s.set_profile(7)
        s.step(pr.n_steps)
        inf = s.info()
        it, _, _ = s.history()
        res.append(inf["prof_ms"])
    s.set_profile(0)
    ms = float(np.median(res))
    print(f"STEP {tag} {name} k_steps {ms:.3f} ms  {1000*ms/pr.n_steps:.1f} us/step  iters/step {np.mean(it):.2f}  "
          f"{1000*ms/np.sum(it):.2f} us/iter(all-in)", flush=True)
    if os.environ.get("REPS"):
        print("   per rep ms:", " ".join(f"{x:.2f}" for x in res))
    s.close()
