"""Shard invariance on one GPU ("per-image outputs bit-identical
across G" is the multi-GPU correctness test).

The batch is split into the contiguous ROI-balanced ranges shard.partition
gives for G = 2, 4, 8 ranks; each range runs on its own plan and its own
stream (what one rank does on its own GPU), all ranges concurrently.  Every
image's output must be bit-identical to the single-plan run of the whole
batch: the kernel has no cross-image state, and tiling / CTA maps chosen per
shard size must not change any value."""
import numpy as np
import pytest
import torch

import paper_2007_13005_b200 as smol
import synth
from paper_2007_13005_b200 import shard

pytestmark = pytest.mark.gpu


def _mixed_batch(name, n):
    cfg = synth.CONFIGS[name]
    imgs, qt = synth.batch_images(cfg, n=n, n_distinct=min(n, 12))
    rng = np.random.default_rng(5)
    extra = []
    for (w, h) in [(333, 500), (97, 61), (640, 480), (161, 161)]:     # heterogeneous sizes
        extra.append(synth.make_image(rng, w, h, qt))
    return cfg, imgs[: n - 4] + extra, qt


@pytest.mark.parametrize("name,n", [("c2", 64), ("c3b", 64), ("c4", 256), ("c5", 12)])
def test_shard_invariance(name, n):
    cfg, imgs, qt = _mixed_batch(name, n)
    ps = smol.params_from_config(cfg, layout="dense" if cfg.scale_denom == 1 else "packed")
    ref_plan = smol.Plan(ps, len(imgs))
    ref = ref_plan.run(smol.batch_for(ps, imgs, qt))
    torch.cuda.synchronize()
    ref = ref.cpu()
    w = shard.roi_weights(ps, imgs)
    for G in (2, 4, 8):
        parts = shard.partition(w, G)
        assert parts[0][0] == 0 and parts[-1][1] == len(imgs)
        outs, keep = [], []
        for lo, hi in parts:
            if hi == lo:
                continue
            plan = smol.Plan(ps, hi - lo)
            s = torch.cuda.Stream()
            b = smol.batch_for(ps, imgs[lo:hi], qt)
            outs.append((lo, hi, plan.run(b, stream=s)))
            keep.append((plan, b, s))
        torch.cuda.synchronize()
        for lo, hi, o in outs:
            assert torch.equal(o.cpu(), ref[lo:hi]), (name, G, lo, hi)
        for plan, _, _ in keep:
            plan.close()
    ref_plan.close()
