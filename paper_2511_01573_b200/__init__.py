"""B200-native h-adaptive cubature (arXiv 2511.01573), drop-in for the
reference package `hcub`'s hot path.

Public names follow ref pkg/src/hcub/__init__.py.  All numerics run in the
sm_100a kernels of libhcub_b200.so (csrc/); Python holds configuration,
host-side protocol decisions and result objects only.
"""

__version__ = "0.1.0"

from ._lib import device_count, set_device, current_device, set_k1_lanes
from .regions import HyperRect, RegionRecord, RegionStore, split, uniform_partition, volume
from .rules import (
    RuleEvaluation,
    RuleTable,
    UnsupportedDimensionError,
    apply_rule,
    apply_rule_batch,
    build_gk_tensor_rule,
    build_gm_rule,
    get_rule,
    load_rule_table,
    parse_rule_table,
    select_axis,
)
from .driver import (
    DriverConfig,
    GlobalEstimate,
    IntegrationResult,
    IterationTrace,
    TerminationReason,
    VolumeBudgetClassifier,
    check_convergence,
    integrate,
)
from .integrands import FUNCTION_IDS, BenchmarkIntegrand, ProductPeak, make_integrand, make_product_peak, reference_integral
from .distributed import (
    BACKENDS,
    DistributedResult,
    MetadataRecord,
    ProtocolError,
    RedistributionConfig,
    TimeBreakdown,
    TransferBatch,
    WorkerState,
    fair_share,
    metadata_reduce,
    plan_transfer,
    round_robin_pairs,
    run_distributed,
)
from .worker import DeviceWorker
from .experiments import ExperimentSpec, SpecError, run_accuracy_sweep, run_idle_breakdown, run_scaling_sweep
