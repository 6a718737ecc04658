"""B200-native stable z-score partitioning sort (zSort, arxiv 2605.14419).

Drop-in for the reference package's sort entry point::

    from paper_2605_14419_b200 import zsort, SortConfig, SortStats
    keys_out, payload_out, stats = zsort(keys, payload, config)

All passes run as hand-written sm_100a CUDA kernels behind the C ABI in
include/zsort_b200.h (libzsort_b200.so, bound with ctypes); see DESIGN.md.
"""

from .core import (  # noqa: F401
    DegenerateSpreadError,
    FirstPassStats,
    MappingParams,
    PartitionPlan,
    SortConfig,
    SortStats,
    all_equal,
    build_mapping_params,
    build_partition_plan,
    check_stable_permutation_device,
    cluster_count,
    estimated_mean,
    counting_sort_stable,
    fallback_sort_stable,
    first_pass,
    insertion_sort_stable,
    map_to_cluster,
    stable_scatter,
    zsort,
    zsort_rec,
)

from .pipeline import SortPipeline  # noqa: F401,E402

__all__ = [
    "SortPipeline",
    "DegenerateSpreadError", "FirstPassStats", "MappingParams", "PartitionPlan", "SortConfig", "SortStats",
    "all_equal", "build_mapping_params", "build_partition_plan", "check_stable_permutation_device",
    "cluster_count", "counting_sort_stable", "estimated_mean", "fallback_sort_stable", "first_pass",
    "insertion_sort_stable", "map_to_cluster", "stable_scatter", "zsort", "zsort_rec",
]
