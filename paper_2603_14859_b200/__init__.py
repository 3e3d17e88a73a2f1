"""paper_2603_14859_b200 -- B200-native voxelwise rejection ABC (vPET-ABC, arxiv 2603.14859).

    ctx = AbcContext(models=[dict(kind="2TCM_IRR", n_draws=N//2, lo=..., hi=...),
                             dict(kind="2TCM_REV", n_draws=N//2, lo=..., hi=...)],
                     seed=2026, distance="WL2", accept="TOPN", n_accept=18)
    ctx.set_input_function("PWL", value=knot_values, t=knot_times)   # or ("FENG", value=beta_kappa)
    ctx.set_frames(start_min, dur_min, weight)
    res = ctx.run_voxels(tacs)      # numpy (host) or torch.cuda tensor (device), J x L float32

The compute runs in libvpetabc.so (CUDA, sm_100a) through the C ABI in include/vpetabc.h.
"""
from ._abi import (AbcError, FLAG_COUNT_WORK, FLAG_DENSE_TC, FLAG_EXACT, FLAG_FORCE_FALLBACK, FLAG_NO_PRUNE, FLAG_NO_REORDER, FLAG_NO_TREE,  # noqa: F401
                   FLAG_TIMING, load_library)
from .context import AbcContext, family_width  # noqa: F401

__all__ = ["AbcContext", "AbcError", "family_width", "load_library", "FLAG_TIMING", "FLAG_EXACT",
           "FLAG_COUNT_WORK", "FLAG_DENSE_TC", "FLAG_FORCE_FALLBACK", "FLAG_NO_PRUNE", "FLAG_NO_REORDER", "FLAG_NO_TREE"]
