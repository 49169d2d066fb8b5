"""Profile driver: C5 (or --config k) batched sweep apply, t directions.
Warm-up applies, then timed applies with CUDA events; prints ms and model GB/s.
Use under ncu with  -k regex:k_sweep_apply -s <warm> -c 1."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_11929_b200 as hs
from helm_inputs import make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--t", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--nseg", type=int, default=0)
ap.add_argument("--names", default="", help="comma-separated directions (overrides --t)")
ap.add_argument("--knob", action="append", default=[], help="name=value (helm_set_knob), repeatable")
a = ap.parse_args()
for kv in a.knob:
    hs.set_knob(kv.split("=")[0], int(kv.split("=")[1]))

cfg = make_config(a.config)
names = a.names.split(",") if a.names else {1: ["LRL"], 2: ["LRL", "BTB"], 4: ["LRL", "RLR", "BTB", "TBT"]}[a.t]
a.t = len(names)
dev = torch.device("cuda:0")
prob = hs.Problem(cfg.nx, cfg.ny, cfg.h, cfg.omega, torch.tensor(cfg.c.ravel(), dtype=torch.float64, device=dev))
dirs = [hs.Sweep(prob, nm, n_strips=cfg.n_strips, overlap=cfg.overlap, n_segments=a.nseg) for nm in names]
info = [d.info() for d in dirs]
r = torch.randn(cfg.n, dtype=torch.complex128, device=dev)
Z = torch.zeros((len(dirs), cfg.n), dtype=torch.complex128, device=dev)
for _ in range(a.warm):
    hs.sweep_apply(dirs, r, Z, ldr=0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    hs.sweep_apply(dirs, r, Z, ldr=0)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
model = sum(i.model_bytes_per_apply for i in info)
print(f"config C{a.config} t={a.t} P={info[0].n_segments} w={info[0].wmax}: {ms:.3f} ms/apply, "
      f"model {model/1e9:.2f} GB -> {model/ms/1e6:.0f} GB/s, applies/s {a.t*1e3/ms:.1f}")

if os.environ.get("HELM_CYCLES"):
    import ctypes
    L = hs.load()
    ctas = sum(i.n_segments + (1 if i.n_segments > 1 else 0) for i in info)  # upper bound
    stride = 32 if hs.sweep_kernel_name() == "k_sweep_dual" else 8
    if stride == 32:
        ctas = sum(i.n_segments for i in info)   # the two-chain kernel: P CTAs per direction
    buf = torch.zeros(ctas * stride + (ctas * 64 if stride == 32 else 0), dtype=torch.int64, device=dev)
    L.helm_sweep_profile.argtypes = [ctypes.c_void_p]
    L.helm_sweep_profile(ctypes.c_void_p(buf.data_ptr()))
    hs.sweep_apply(dirs, r, Z, ldr=0)
    torch.cuda.synchronize()
    L.helm_sweep_profile(ctypes.c_void_p(0))
    b = buf[:ctas * stride].view(ctas, stride).cpu().numpy()
    if stride == 32 and os.environ.get("HELM_SKEW"):
        import numpy as np
        gt = buf[ctas * stride:].view(ctas, 64).cpu().numpy().astype(np.float64)
        P = info[0].n_segments
        ns = 63
        for d in range(len(info)):
            g = gt[d * P:(d + 1) * P, :ns]
            late = g - g.min(axis=0, keepdims=True)       # ns behind the first CTA of the direction
            print(f"  dir {d}: phase-1 end skew per solve (ns): mean max {late.max(axis=0).mean():.0f}, "
                  f"mean {late.mean():.0f}; latest CTA counts: " +
                  " ".join(f"{p}:{c}" for p, c in sorted(((p, int((late.argmax(axis=0) == p).sum())) for p in range(P)), key=lambda x: -x[1])[:6]))
            print(f"    mean lateness by segment (ns): " + " ".join(f"{v:.0f}" for v in late.mean(axis=1)))
    if stride == 32:
        sel = b[b[:, 3] > 0]
        tp = sel[:, 8:12].mean(axis=0) / sel[:, 3].mean()
        print(f"  dual step sub-phases (cycles/step, thread 0): mat-vec {tp[0]:.0f}  loads+reduce+nb {tp[1]:.0f}  "
              f"writer {tp[2]:.0f}  barrier {tp[3]:.0f}")
        ns = sel[:, 3].mean() / (2 * 31)
        print(f"  separator stage per solve (cycles, thread 0): gather wait {sel[:,12].mean()/63:.0f}  "
              f"corrections+g {sel[:,14].mean()/63:.0f}  X mat-vec {sel[:,2].mean()/63:.0f}  neighbour wait {sel[:,13].mean()/63:.0f}  "
              f"total {sel[:,1].mean()/63:.0f};  pre-actions {sel[:,0].mean()/63:.0f}")
        print(f"  balanced separator stage (thread 0, per solve): pass A {sel[:,15].mean()/63:.0f}  pass B {sel[:,11].mean()/63:.0f}")
        print(f"  pre-actions (thread 0, per solve): other group's tail {sel[:,9].mean()/63:.0f}  through epilogue {sel[:,10].mean()/63:.0f}  "
              f"coupling wait (slot 15) {sel[:,15].mean()/63:.0f}  stage_bands issue {sel[:,22].mean()/63:.0f}  +staging waits {sel[:,23].mean()/63:.0f}")
        print(f"  pre-action tail (thread 0, per solve): seg_rhs {sel[:,27].mean()/63:.0f}  +source staging issue {sel[:,28].mean()/63:.0f}  "
              f"+barrier {sel[:,29].mean()/63:.0f}")
        P0 = info[0].n_segments
        d0 = b[:P0]
        print("  two-level per CTA of direction 0 (per solve): wait coarse / round 1 / round 2: " +
              " ".join(f"{p}:{d0[p,24]/63:.0f}/{d0[p,25]/63:.0f}/{d0[p,26]/63:.0f}" for p in range(P0)))
        print(f"  phases (thread 0, per solve): phase 1 {sel[:,19].mean()/63:.0f}  phase 3 {sel[:,20].mean()/63:.0f}  stage_next {sel[:,21].mean()/63:.0f} | "
              f"separator stage: yb {sel[:,16].mean()/63:.0f}  X+publish {sel[:,17].mean()/63:.0f}  x_lo+inputs {sel[:,18].mean()/63:.0f}")
    for role in (0, 1):
        sel = b[b[:, 6] == role]
        if len(sel) == 0:
            continue
        sel = sel[sel[:, 3] > 0]
        st = sel[:, 3].mean()
        print(f"  totals per CTA: pre(epilogue+rhs) {sel[:,0].mean():.3e}  sep-stage {sel[:,1].mean():.3e}  "
              f"slot2 (warp: ring wait, dual: X mat-vec) {sel[:,2].mean():.3e}  xwait {sel[:,4].mean():.3e}  "
              f"steps {(sel[:,5]-sel[:,0]-sel[:,1]).mean():.3e} -> {(sel[:,5]-sel[:,0]-sel[:,1]).mean()/st:.0f} cyc/step")
        print(f"{'reducer' if role else 'segment'} CTAs={len(sel)} steps={st:.0f} total={sel[:,5].mean():.3e} cyc | "
              f"per step: pre|peek {sel[:,0].mean()/st:.0f} comp {sel[:,1].mean()/st:.0f} bar {sel[:,2].mean()/st:.0f} | "
              f"xwait total {sel[:,4].mean():.3e} ({sel[:,4].mean()/sel[:,5].mean()*100:.1f}%) | "
              f"X mat-vec total {sel[:,7].mean():.3e} ({sel[:,7].mean()/sel[:,5].mean()*100:.1f}%)")
