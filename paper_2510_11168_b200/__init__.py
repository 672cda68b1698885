"""B200-native ELMO extreme-classification head (arxiv 2510.11168).

Drop-in for the reference package's hot path (lpxmc.head / lpxmc.optimizers /
lpxmc.formats): same names and semantics on torch CUDA tensors, computed by
hand-written sm_100a kernels (libxmc_b200.so, C ABI in include/xmc_head.h).
"""

from .formats import (BF16, E4M3, E5M2, FP16, FP32, FloatFormat, RoundingRng, parse_format,
                      round_nearest, round_stochastic, tensor_tag)
from .optimizers import (KahanAdamWConfig, KahanAdamWParam, SgdSrConfig, kahan_adamw_step, kahan_sgd_step,
                         sgd_sr_step)
from .head import (DROPOUT_TAG, HEAD_WEIGHTS_TAG, N_CELLS, BatchInput, ChunkedHead, QuantizedMatrix,
                   canonical_pieces, cast_native, dropout_mask, fused_weight_update, head_forward_logits,
                   head_update, input_gradient_accumulate, load_head, logit_gradient, partition,
                   save_head)

from . import metrics, trainer_hooks

__version__ = "0.2.0"
