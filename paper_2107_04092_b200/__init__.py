"""B200-native (sm_100a) clock-driven SNN step of arXiv 2107.04092 ("Spice"):
lazy + event-driven STDP over 64-bit spike bitfields and neuron-domain-sliced
spike delivery with shared-memory atomics, behind the C ABI of include/snn.h.

``from paper_2107_04092_b200 import Snn`` loads libsnn.so (built by
``__graft_entry__.build()``) and raises if it is missing -- there is no CPU
fallback on the product path.
"""
from .snn import *  # noqa: F401,F403
from .snn import Snn, SnnError, EXPORTS, LIB_PATH  # noqa: F401
