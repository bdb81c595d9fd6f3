"""atk-b200: B200-native (sm_100a) generalized two-stage approximate top-k
(arXiv 2506.04165), a drop-in for the reference `atk` core hot path.

The compute runs in libatkg.so (hand-written CUDA for sm_100a behind the C ABI
in include/atkg.h); this package is the host-side mirror of the reference
interface.  Importing fails loudly if the library has not been built.
"""
from ._lib import NoFeasibleConfigError  # noqa: F401
from .mips import (MipsResult, MipsStats, default_block_cols, mips_fused, mips_unfused,  # noqa: F401
                   validate_mips_request)
from .simulate import (SimStats, simulate_recall, simulate_recall_many, synth_distinct,  # noqa: F401
                       synth_distinct_device, synth_distinct_row)
from .dataset import (DatasetFormatError, VectorDataset, read_dataset_file, read_dataset_to_device,  # noqa: F401
                      write_dataset_file, write_dataset_from_device)
from .planner import (PlanRequest, PlanResult, RecallEstimate, approx_top_k_at_recall, exact_expected_recall,  # noqa: F401
                      legal_bucket_counts, mc_expected_recall, mc_expected_recall_adaptive,
                      select_parameters)
from .topk import (AlgoParams, Stage1Accumulator, TopKResult, approx_top_k, approx_top_k_batch, check_status,  # noqa: F401
                   approx_top_k_device, exact_top_k, exact_top_k_device, kDefaultLaneMultiple, kNegInf,
                   measure_recall, partition_index, select_candidates_device, select_top_k_candidates,
                   stage1_device, stage1_partial_reduce, stage1_summary_device, summary_merge_top_k_device,
                   summary_words, slice_payload_words, slice_payload_device, payload_merge_top_k_device,
                   NcclComm, sharded_approx_top_k_device)

__version__ = "0.1.0"
