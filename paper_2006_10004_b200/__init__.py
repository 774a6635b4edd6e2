"""B200-native TVSpecNET inference (arXiv 2006.10004) — drop-in for the
reference ``tvsurrogate.model`` module, backed by libtvsb200.so (sm_100a).

Public surface mirrors /root/reference/pkg/trainer/src/tvsurrogate:
``TVSpecNet``, ``ARCH_SPEC``, ``receptive_field`` (model.py) and
``predict_bands``, ``complete_planes``, ``bench_forward`` (inference.py).
"""

from .model import ARCH_SPEC, TVSpecNet, receptive_field
from .inference import bench_forward, complete_planes, predict_bands, predict_planes

__all__ = [
    "ARCH_SPEC",
    "TVSpecNet",
    "receptive_field",
    "predict_bands",
    "predict_planes",
    "complete_planes",
    "bench_forward",
]

__version__ = "0.1.0"
