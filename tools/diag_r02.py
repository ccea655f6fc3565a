"""Round-2 diagnosis (GPU): per-tensor errors of (a) the 1-sample BN tail fixture, (b) C1 fp32 variants."""
import copy
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2110_12484_b200 as mbs  # noqa: E402
from paper_2110_12484_b200 import bn as K5, engine, graphs  # noqa: E402
from tests.golden_io import load_json, load_npz  # noqa: E402
from tests.refmodels import build_torch, load_ref_params, to_ref  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
cuda = torch.device("cuda:0")


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n else float(np.linalg.norm(a - b))


def bn1():
    name = "bn1_tail"
    meta = load_json("e2e.json")[name]
    a = load_npz("e2e.npz")
    for graphs_on in (True, False):
        engine.CUDA_GRAPHS = graphs_on
        graphs.clear()
        for mode in ("exact_weighted", "off"):
            torch.manual_seed(0)
            mod = build_torch(meta["spec"], tuple(meta["input_shape"])).to(cuda)
            load_ref_params(mod, meta["spec"], {n: a[f"{name}/p0/{n}"] for n in meta["param_names"]})
            K5.fuse_batchnorm(mod)
            params = mbs.ParameterSet(mod)
            x = torch.from_numpy(a[f"{name}/x"][:9]).float().to(cuda)
            y = torch.from_numpy(a[f"{name}/y"][:9]).to(cuda)
            total, st = mbs.mini_batch_gradient(mod, params, x, y, mbs.plan_split(9, 4), mode, "cross_entropy")
            got = to_ref(meta["spec"], {tn: total[tn] for tn in params.names()})
            print("bn1", "graphs" if graphs_on else "eager", mode,
                  {k: round(rel(got[k], a[f"{name}/{mode}/grad0/{k}"]), 8) for k in sorted(got)})
            # per micro: single-micro gradients vs torch-fp64 with biased-var BN written out
    engine.CUDA_GRAPHS = True


def c1_variants():
    from oracle import mbs_oracle as O
    from oracle.hybrid import TorchGradFn
    from paper_2110_12484_b200.streamer import Staging
    from paper_2110_12484_b200.workloads import WORKLOADS, build_model, make_native
    w = WORKLOADS["c1"]
    torch.manual_seed(0)
    net = build_model(w, ops="torch").train()
    g = torch.Generator().manual_seed(11)
    x = torch.randint(0, 256, (64, 3, 32, 32), dtype=torch.uint8, generator=g)
    y = torch.randint(0, 10, (64,), generator=g)
    plan = O.plan_split(64, 8)
    ref = TorchGradFn(net, w.loss_kind)
    names = ref.names
    g64, _ = O.mini_batch_gradient(ref, {n: v.shape for n, v in ref.params().items()}, x.double().numpy(),
                                   y.numpy(), plan, w.normalization)
    flat64 = np.concatenate([g64[n].ravel() for n in names])

    def swap(m, which):
        from paper_2110_12484_b200.pool import swap_maxpool
        from paper_2110_12484_b200.stem import swap_pointwise, swap_stem
        if "k5" in which:
            K5.fuse_batchnorm(m)
        if "k6" in which:
            swap_maxpool(m)
        if "k7" in which:
            swap_stem(m)
            swap_pointwise(m)
        return m

    out = {}
    for which in ("none", "k5", "k6", "k7", "k5k6k7"):
        for staged in (True, False):
            for graphs_on in (True, False):
                engine.CUDA_GRAPHS = graphs_on
                graphs.clear()
                dnet = swap(copy.deepcopy(net), which).to(cuda).to(memory_format=torch.channels_last)
                params = mbs.ParameterSet(dnet)
                if staged:
                    xs, st_ = x.to(cuda), Staging(torch.float32, True)
                else:
                    xs, st_ = x.float().to(cuda).contiguous(memory_format=torch.channels_last), None
                total, _ = mbs.mini_batch_gradient(dnet, params, xs, y.to(cuda), mbs.plan_split(64, 8),
                                                   w.normalization, w.loss_kind, staging=st_)
                got = np.concatenate([total[n].detach().double().cpu().numpy().ravel() for n in names])
                key = f"{which}/{'staged' if staged else 'f32in'}/{'graph' if graphs_on else 'eager'}"
                out[key] = rel(got, flat64)
                print("c1fp32", key, out[key], flush=True)
    engine.CUDA_GRAPHS = True
    # plain
    pnet = copy.deepcopy(net).to(cuda).to(memory_format=torch.channels_last)
    for k, (lo, hi) in enumerate(plan.index_ranges):
        f = O.normalization_factor(plan, k, w.normalization)
        (mbs.compute_loss(w.loss_kind, pnet(x[lo:hi].float().to(cuda).contiguous(memory_format=torch.channels_last)),
                          y[lo:hi].to(cuda)) * f).backward()
    plain = np.concatenate([dict(pnet.named_parameters())[n].grad.double().cpu().numpy().ravel() for n in names])
    out["plain"] = rel(plain, flat64)
    print("c1fp32 plain", out["plain"])
    with open(os.path.join(ROOT, "gpurun_out", "diag_r02.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    bn1()
    c1_variants()
