"""B200-native HOOI engine for dense Tucker decomposition (hot path of arXiv 1707.05594's
`tuckerplan` reference): host-side mirror of the reference API over the C ABI in
include/tuckerplan_b200.h.  PyTorch is not needed to use the engine."""
from ._lib import Errc, TuckerplanError, lib, LIB_PATH  # noqa: F401
from . import planner  # noqa: F401
