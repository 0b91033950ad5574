"""splitgnn-b200: B200-native split-parallel GNN training step (arXiv 2303.13775).

Drop-in for the reference `splitgnn` package's hot path: same public names
(sample_minibatch, split_minibatch, SplitExecutor, allreduce_and_step,
init_params, ...), backed by the sm_100a library libsplitgnn_b200.so through
the C ABI in include/splitgnn_b200.h. There is no CPU fallback.
"""

from paper_2303_13775_b200.graph import (
    Graph,
    GraphError,
    from_edges,
    generate_powerlaw,
    load_binary_csr,
    save_binary_csr,
    synthetic_features,
    synthetic_labels,
)
from paper_2303_13775_b200.partition import (
    CacheState,
    PartitionMap,
    build_cache,
    cut_size,
    full_cache,
    max_part_size,
    partition_graph,
    range_partition,
    refine_assignment,
)
from paper_2303_13775_b200.sampling import (GpuSampler, MiniBatchSample, NativeSampler, epoch_batches,
                                            sample_microbatches, sample_minibatch)
from paper_2303_13775_b200.scheduler import (
    DeviceSplit,
    LocalSplit,
    PlanEntry,
    ShufflePlan,
    SplitCostReport,
    split_cost,
    split_minibatch,
    transfer_manifest,
)
from paper_2303_13775_b200.models import DeviceParams, GatLayer, ModelParams, SageLayer, init_params
from paper_2303_13775_b200.metrics import (EpochMetrics, IterationMetrics, account_transfer, emit_csv, read_csv,
                                           redundancy_report, union_edge_count)
from paper_2303_13775_b200.features import FeatureStore
from paper_2303_13775_b200.exchange import (LocalTransport, NcclTransport, PeerTransport, exchange_microbench,
                                            uniform_exchange_sample)
from paper_2303_13775_b200.engine import (
    PhaseRunner,
    SplitExecutor,
    SplitStep,
    Trainer,
    allreduce_and_step,
    scatter_shuffle_forward,
    train_model,
)

__all__ = [n for n in dir() if not n.startswith("_")]
