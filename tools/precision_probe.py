"""Per-stage error budget of the fp32 path against the float64 torch.fft
restatement (oracle/torch_ref.py): cached pre-activations, y, and for the
mixer weight gradients the split between the kernel's own error (float64
product of OUR cached operands) and the propagated forward error.

  python tools/precision_probe.py --grid 64,64,64,32 --c 20 --blocks 4 [--ranks P]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2211_12709_b200 as P  # noqa: E402
from oracle import torch_ref as R  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="64,64,64,32")
    ap.add_argument("--modes", default="8,8,8,8")
    ap.add_argument("--c", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=4)
    ap.add_argument("--act", default="gelu")
    ap.add_argument("--gy", action="store_true", help="g = y instead of a random g")
    ap.add_argument("--seed", type=int, default=22)
    args = ap.parse_args()
    grid = tuple(int(v) for v in args.grid.split(","))
    modes = tuple(int(v) for v in args.modes.split(","))
    config = P.FnoConfig(*grid, args.c, args.c, args.c, P.ModeSpec.of_xyzt(*modes), args.blocks, args.act,
                         "real32", 1)
    dev = torch.device("cuda")
    params = P.init_params(config, args.seed, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed)
    x = torch.randn((1, args.c) + grid, generator=gen, device=dev)
    g = torch.randn((1, args.c) + grid, generator=gen, device=dev)

    out = {}

    def body(comm):
        cache = P.ForwardCache()
        y = P.fno_forward(comm, P.DenseTensor(P.DATA_LABELS, x), params, config, cache=cache)
        gg = y if args.gy else P.DenseTensor(P.DATA_LABELS, g)
        gx, grads = P.fno_backward(comm, gg, params, config, cache)
        return y.data, gx.data, grads, cache

    y, gx, grads, cache = P.run_ranks(1, body)[0]
    blocks = [w.data for w in params.blocks]
    ry, rc = R.forward(x, params.we.data, params.wd.data, blocks, modes, args.act)
    out["enc_pre"] = R.rel_err(cache.enc_pre.data, rc["enc_pre"])
    for i, b in enumerate(cache.blocks):
        out[f"pre{i}"] = R.rel_err(b.pre_activation.data, rc["pres"][i])
        out[f"spec{i}"] = R.rel_err(b.spec_in.data, rc["specs"][i])
    out["dec_pre"] = R.rel_err(cache.dec_pre.data, rc["dec_pre"])
    out["y"] = R.rel_err(y, ry)
    gref = ry if args.gy else g.double()
    # gWd from OUR cached operands in float64: isolates the kernel's own error
    a_last = R.act(args.act, cache.blocks[-1].pre_activation.data.double())
    gd = (y.double() if args.gy else g.double()) * R.act_grad(args.act, cache.dec_pre.data.double())
    gwd_ours64 = R.mix_weight_grad(a_last, gd)
    out["gwd_kernel_only"] = R.rel_err(grads.wd.data, gwd_ours64)
    del a_last, gd
    rgx, rgwe, rgwd, rgws = R.backward(gref, params.we.data, params.wd.data, blocks, modes, rc, args.act)
    out["gwd_forward_propagated"] = R.rel_err(gwd_ours64, rgwd)
    out["gwd"] = R.rel_err(grads.wd.data, rgwd)
    out["gwe"] = R.rel_err(grads.we.data, rgwe)
    out["gx"] = R.rel_err(gx, rgx)
    for i, gw in enumerate(grads.blocks):
        out[f"gw{i}"] = R.rel_err(gw.data, rgws[i])
    # magnitudes: how much the random-g mixer gradients cancel
    out["gwd_abs_max"] = rgwd.abs().max().item()
    print(json.dumps({k: (f"{v:.3e}" if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
