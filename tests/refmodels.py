"""Torch modules equivalent to the reference's ModelSpec layer stacks (nn.py:33-73, 130-410).

Test infrastructure: maps a golden fixture's spec + reference-named parameters
onto a torch module and back, so the B200 path can be checked against the
reference's own outputs. Dense weights are stored (in, out) by the reference
(nn.py:141) and (out, in) by torch.
"""
import numpy as np
import torch
from torch import nn


def build_torch(spec, input_shape):
    layers, names = [], []
    rank = len(input_shape)
    for i, e in enumerate(spec):
        t = e["type"]
        if t == "Dense":
            layers.append(nn.Linear(e["in_features"], e["out_features"], bias=e["bias"]))
        elif t == "Conv2d":
            layers.append(nn.Conv2d(e["in_channels"], e["out_channels"], e["kernel"], e["stride"], e["padding"]))
        elif t == "Relu":
            layers.append(nn.ReLU())
        elif t == "BatchNorm":
            bn = nn.BatchNorm2d if rank == 3 else nn.BatchNorm1d
            layers.append(bn(e["features"], eps=e["epsilon"], momentum=e["momentum"]))
        elif t == "Flatten":
            layers.append(nn.Flatten())
            rank = 1
        elif t == "MaxPool2d":
            layers.append(nn.MaxPool2d(e["kernel"], e["stride"] if e["stride"] is not None else e["kernel"]))
        else:
            raise ValueError(t)
        names.append(t)
    return nn.Sequential(*layers)


def name_map(spec):
    """reference name -> (torch name, transpose?)"""
    out = {}
    for i, e in enumerate(spec):
        t = e["type"]
        if t == "Dense":
            out[f"layer{i}.weight"] = (f"{i}.weight", True)
            if e["bias"]:
                out[f"layer{i}.bias"] = (f"{i}.bias", False)
        elif t == "Conv2d":
            out[f"layer{i}.weight"] = (f"{i}.weight", False)
            out[f"layer{i}.bias"] = (f"{i}.bias", False)
        elif t == "BatchNorm":
            out[f"layer{i}.gamma"] = (f"{i}.weight", False)
            out[f"layer{i}.beta"] = (f"{i}.bias", False)
    return out


def load_ref_params(module, spec, ref_params: dict):
    nm = name_map(spec)
    sd = dict(module.named_parameters())
    with torch.no_grad():
        for rname, (tname, tr) in nm.items():
            v = np.asarray(ref_params[rname])
            v = v.T if tr else v
            sd[tname].copy_(torch.from_numpy(np.ascontiguousarray(v)).to(sd[tname].dtype))


def to_ref(spec, torch_dict: dict) -> dict:
    """torch-named tensors/arrays -> reference-named float64 arrays."""
    out = {}
    for rname, (tname, tr) in name_map(spec).items():
        v = torch_dict[tname]
        v = v.detach().double().cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, np.float64)
        out[rname] = v.T if tr else v
    return out
