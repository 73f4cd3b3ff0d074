"""B200-native Fastfood (McKernel, arXiv 1702.08159) hot path.

Drop-in for the reference package's hot path (``mckernel`` 0.1.0,
``pkg/src/mckernel/__init__.py:7-56``): the names below keep the reference's
signatures; the work runs in the sm_100a library ``libmckernel_b200.so``
through the C ABI declared in ``include/mckernel_b200.h``.
"""

__version__ = "0.1.0"

from .fastfood import (
    RBF,
    BlockSet,
    FastfoodBlock,
    FeatureMapSpec,
    RBFMatern,
    apply_zhat,
    apply_zhat_batch,
    blocks_from_reference,
    build_block,
    build_blocks,
    feature_dim,
    feature_map,
    feature_map_batch,
    next_pow2,
    param_count,
)
from .wht import is_power_of_two, wht_fast, wht_fast_batch
from .detrand import RandomStream, fisher_yates_permutation, fisher_yates_permutations
from .linear_model import (
    Dataset,
    EpochRecord,
    RunMetrics,
    SoftmaxModel,
    TrainConfig,
    Trainer,
    evaluate,
    forward,
    forward_batch,
    gradients,
    loss,
    sgd_step,
    train,
)

__all__ = [
    "RBF", "RBFMatern", "FeatureMapSpec", "FastfoodBlock", "BlockSet", "next_pow2",
    "build_block", "build_blocks", "blocks_from_reference", "apply_zhat", "apply_zhat_batch",
    "feature_map", "feature_map_batch", "feature_dim", "param_count",
    "wht_fast", "wht_fast_batch", "is_power_of_two",
    "RandomStream", "fisher_yates_permutation", "fisher_yates_permutations",
    "Dataset", "EpochRecord", "RunMetrics", "SoftmaxModel", "TrainConfig", "Trainer",
    "evaluate", "forward", "forward_batch", "gradients", "loss", "sgd_step", "train",
]
