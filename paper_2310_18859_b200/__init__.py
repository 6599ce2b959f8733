"""SiDA data-aware MoE serving hot path, B200-native (sm_100a).

Public names mirror the hot-path subset of the reference package's API
(ref pkg/src/sida/__init__.py:1-50): the hash-function predictor, the
expert hash table, the FIFO residency planner and the two-worker serving
loop. Compute runs in the hand-written CUDA library `_sida_b200.so`
(include/sida_b200.h); there is no CPU fallback.
"""

from .errors import ContractError, CoverageError, NativeLibraryError, TrainingDiverged, UnservableError
from .moe import (
    ActivationTrace,
    BatchLayout,
    MoEConfig,
    MoEModel,
    Rng,
    SequenceBatch,
    model_forward,
    moe_layer_forward,
    router_scores,
)
from .numkit import check_finite, softmax, sparsemax, topk, topk_rows
from .predictor import (
    DeviceTable,
    ExpertHashTable,
    PredictorConfig,
    OracleHasher,
    PredictorHasher,
    PredictorNet,
    build_hash_table,
    hash_hit_rate,
)
from .offload import (
    ExpertStore,
    MemoryBudget,
    PlacementPlan,
    PlanGroup,
    ResidencyState,
    apply_group_inplace,
    apply_plan,
    effective_utilization,
    ensure_layer_resident,
    memory_reduction,
    plan_placement,
)
from .checkpoint import load_moe, load_predictor, save_moe, save_predictor
from .pipeline import HashTableQueue, ServingReport, fidelity, serve_sida, serve_standard

__version__ = "0.1.0"
