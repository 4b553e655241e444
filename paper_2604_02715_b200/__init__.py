"""B200-native expert-paging MoE layer (drop-in for the hot path of FluxMoE's ``xpg``).

PagedTensor-backed expert weights in an HBM ring, a per-layer page-in/evict
schedule on CUDA copy streams, and a MoE forward (hash router, expert-major
permute, tcgen05 grouped SwiGLU GEMMs, ordered combine) — all hand-written
sm_100a CUDA in ``libxpgb.so`` behind the C ABI of ``include/xpgb.h``.  The
Python names mirror the reference package (xpg/__init__.py:10-39) for the
paged path.
"""

from .errors import (
    BackendMissError,
    CapacityExceededError,
    ConfigError,
    ContainerFormatError,
    DeadlockError,
    DoubleMapError,
    InfeasibleConfigError,
    NotMappedError,
    OutOfRangeError,
    PageFaultError,
    PoolExhaustedError,
    XpgError,
)
from .geometry import (
    ExpertTensorId,
    ModelSpec,
    SharedExperts,
    TensorKind,
    WeightContainer,
    bf16_to_float32,
    float32_to_bf16,
    generate_fast_model,
    generate_synthetic_model,
    initial_activations,
    iter_tensor_ids,
    open_container,
    tensor_offset,
)
from .pagetable import AddressSpace, PageState, PageTable, page_vaddr, target_layer
from .tiers import Backend, BackendKind, PlacementPlan, StorageHierarchy, estimate_load, plan_placement
from .streamed import (
    ForwardSpec,
    OrderingRecord,
    ResidentModel,
    RunReport,
    StreamedRunner,
    layer_forward,
    resident_baseline,
    routed_experts,
    run_iterations,
    validate_ordering,
)

__version__ = "0.1.0"
