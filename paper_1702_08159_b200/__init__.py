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
    spec_from_config,
    spec_to_config,
)
from .wht import BenchRecord, bench_wht, bench_wht_csv, is_power_of_two, wht_fast, wht_fast_batch, wht_naive
from .exact_kernel import KernelCheckStats, kernel_check, rbf_kernel
from .dataio import features_to_file, read_matrix, write_matrix
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
    load_model,
    loss,
    save_model,
    sgd_step,
    train,
)
from .large_scale import FusedClassifier

__all__ = [
    "RBF", "RBFMatern", "FeatureMapSpec", "FastfoodBlock", "BlockSet", "next_pow2",
    "build_block", "build_blocks", "blocks_from_reference", "apply_zhat", "apply_zhat_batch",
    "feature_map", "feature_map_batch", "feature_dim", "param_count",
    "spec_to_config", "spec_from_config",
    "wht_fast", "wht_fast_batch", "wht_naive", "is_power_of_two", "bench_wht", "bench_wht_csv", "BenchRecord",
    "kernel_check", "rbf_kernel", "KernelCheckStats",
    "features_to_file", "read_matrix", "write_matrix", "save_model", "load_model",
    "FusedClassifier",
    "RandomStream", "fisher_yates_permutation", "fisher_yates_permutations",
    "Dataset", "EpochRecord", "RunMetrics", "SoftmaxModel", "TrainConfig", "Trainer",
    "evaluate", "forward", "forward_batch", "gradients", "loss", "sgd_step", "train",
]
