"""B200 (sm_100a) implementation of GAPA's data-parallel hot path behind the reference's
operator API.  Compute goes through the C ABI in include/gapa_cuda.h
(paper_2412_20980_b200/libgapa_cuda.so); there is no CPU fallback."""
from . import api, capi, experiment  # noqa: F401
from .api import *  # noqa: F401,F403
