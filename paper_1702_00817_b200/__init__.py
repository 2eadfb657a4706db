"""B200-native blockwise 8x8 approximate DCT (arxiv 1702.00817).

Drop-in for the hot path of the reference package `adct`: the codec and
metric functions keep their names and signatures (codec.py:24-155,
metrics.py:24-97) and run on sm_100a kernels in libadct_cuda.so through a C
ABI (include/adct_cuda.h).  The batched device API lives in `batch`,
multi-GPU sharding in `shard`, the host-buffer pipeline in `pipeline`, the
GPU-backed corpus sweep in `sweep`, PGM ingestion in `pgm`.
"""

from .codec import (
    ZIGZAG_INDICES,
    coefficient_blocks,
    compress_image,
    compression_ratio,
    fold_scaling_into_quantization,
    forward_2d,
    forward_2d_unscaled,
    inverse_2d,
    reconstruct_image,
    retain_coefficients,
    retention_mask,
    zigzag_positions,
)
from .errors import (
    BadDimensions,
    DimensionMismatch,
    DuplicateName,
    EmptyGroup,
    InvalidRetention,
    IoFailure,
    MalformedHeader,
    MissingImage,
    NonOrthogonalKernel,
    NonPositiveQuantizer,
    TruncatedData,
    UnsupportedMaxval,
    UnsupportedQuantizer,
    ZeroRow,
)
from .flowgraph import OpCount, count_operations, fast_forward, flow_intermediates
from .metrics import CorpusSummary, QualityRecord, ape_vs_dct, mse, psnr, summarize
from .sweep import ExperimentConfig, compare_transforms, load_corpus_images, resolve_transform, run_sweep, write_sweep_outputs
from .transforms import (
    ApproximateTransform,
    DiagonalScaling,
    ExactDct,
    TransformMatrix,
    exact_dct_matrix,
    proposed_kernel,
    proposed_scaling,
    proposed_transform,
    stage_matrices,
)

__version__ = "1.0.0"
