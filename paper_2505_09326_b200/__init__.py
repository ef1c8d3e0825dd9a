"""B200-native FlashSign: the spherical-attention forward of arxiv 2505.09326 as
an sm_100a tcgen05/TMEM/TMA kernel behind the reference's ``ncstream`` API.

Layout:
  csrc/            CUDA kernel + host launcher + C-ABI (include/flashsign.h)
  _lib.py          ctypes binding of the C-ABI (libflashsign.so, built in-tree)
  flashsign.py     torch-native entry: fwd(q, k, v) on BSHD CUDA tensors
  attention.py     drop-in ncstream.attention API (numpy / DenseTensor in, out)
  normalizers.py   NormalizerSpec / SPHERICAL / DegenerateDenominatorError
  tensor.py        DenseTensor / ShapeMismatchError / allclose
  partition.py     batch x head sharding across GPUs (one process per GPU)
  pipeline.py      host-resident inputs: chunked H2D / compute / D2H overlap
"""

from ._errors import ConfigError
from .attention import (
    AttentionConfig,
    ScoreBufferMeter,
    TileConfig,
    apply_multiplicity,
    apply_multiplicity_array,
    default_score_scale,
    get_compute_dtype,
    multi_head_attention,
    multi_head_attention_array,
    naive_attention_array,
    naive_generalized_attention,
    set_compute_dtype,
    streamed_attention,
    streamed_attention_array,
)
from .normalizers import SIGNED_L1, SOFTMAX, SPHERICAL, DegenerateDenominatorError, NormalizerSpec, get_spec
from .tensor import CloseReport, DenseTensor, ShapeMismatchError, allclose, quantize_f16_array

__version__ = "0.1.0"
