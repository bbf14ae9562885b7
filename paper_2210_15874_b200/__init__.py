"""B200-native bucket-elimination engine for QAOA MaxCut lightcones.

Drop-in for the hot path of the reference `qtnsim` package
(/root/reference/pkg/src/qtnsim/__init__.py:4-42): the same names for the
circuit / network builders, the ordering + dry-run planner and the
bucket-elimination calls, with every bucket contracted by hand-written
sm_100a kernels (csrc/qtn_b200.cu) behind a C ABI (include/qtn_b200.h).
"""
from .circuits import (
    Circuit,
    Gate,
    Graph,
    QaoaParams,
    gate_diagonal,
    gate_unitary,
    parse_circuit,
    parse_graph,
    qaoa_maxcut_circuit,
    random_regular_graph,
    read_circuit,
    read_graph,
)
from .tensor_core import (
    Backend,
    Bucket,
    BucketStats,
    DeviceTensor,
    Tensor,
    contract_bucket,
    memory_estimate,
    permute,
    process_bucket,
)
from .tn_build import (
    Lightcone,
    TensorNetwork,
    amplitude_network,
    cone_gates,
    extract_lightcone,
    qaoa_energy,
    qaoa_energy_detailed,
    tight_cone_gates,
    zz_sandwich_network,
)
from .ordering import (
    MemoryCapError,
    WidthProfile,
    contract_network,
    contract_network_eager,
    contract_sliced,
    dry_run,
    get_result_data,
    greedy_order,
    line_graph,
    slice_network,
    suggest_slicing,
    write_width_profile_csv,
)
from ._native import NativeError, NativeUnavailable

__all__ = [
    "Backend", "Bucket", "BucketStats", "Circuit", "DeviceTensor", "Gate", "Graph",
    "Lightcone", "MemoryCapError", "NativeError", "NativeUnavailable", "QaoaParams",
    "Tensor", "TensorNetwork", "WidthProfile", "amplitude_network", "cone_gates",
    "contract_bucket", "contract_network", "contract_network_eager", "contract_sliced", "dry_run",
    "extract_lightcone", "gate_diagonal", "gate_unitary", "get_result_data",
    "greedy_order", "line_graph", "memory_estimate", "parse_circuit", "parse_graph",
    "permute", "process_bucket", "qaoa_energy", "qaoa_energy_detailed",
    "qaoa_maxcut_circuit", "random_regular_graph", "read_circuit", "read_graph",
    "slice_network", "suggest_slicing", "tight_cone_gates", "write_width_profile_csv",
    "zz_sandwich_network",
]

__version__ = "0.1.0"
