"""B200-native factored Levenberg-Marquardt registration hot path.

Drop-in for the per-iteration path of the reference ``warplm`` library
(arxiv/paper_2603_19371): trilinear warp + LNCC loss/gradient + rank-1 LM
step + Gaussian smoothing + compositive resample + device-side trust-region
damping and rejection, as hand-written sm_100a CUDA kernels behind the C-ABI
in include/wlm.h.  This package is a thin ctypes layer over that library;
there is no CPU fallback.
"""
from ._lib import LIB_PATH, load  # noqa: F401
from .warplm import *  # noqa: F401,F403
from .warplm import Context, default_context, reg_config  # noqa: F401
from .engine import BatchPipeline, Engine, SlabGroup  # noqa: F401

__version__ = "0.1.0"
