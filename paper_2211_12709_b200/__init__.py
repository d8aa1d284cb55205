"""B200-native domain-decomposed 4-D Fourier neural operator (arXiv 2211.12709).

Drop-in for the hot path of the reference package ``distfno``
(/root/reference/pkg/src/distfno/__init__.py:8-62): the model layer
(config, params, forward / backward, caches, gradients), the partition and
repartition objects, the collectives with exact accounting, and the labelled
tensor and spectral helpers -- computed by the sm_100a kernels of
``lib/libdfno.so`` (C ABI: include/dfno.h) on CUDA, with NCCL carrying the
x <-> ky repartitions between GPUs.  Out of scope (not on the FNO path):
the task pool, the CLI and the
socket transport.  The training step (train_step, Adam) -- the
first caller of the path -- runs on device kernels too.
"""

from .comm import (
    CommStats,
    Communicator,
    PrimitiveStats,
    ProcessGroupBackend,
    ThreadWorld,
    aggregate_stats,
    comm_report,
    run_ranks,
)
from .errors import (
    CollectiveMismatchError,
    CollectiveTimeoutError,
    DimensionMismatchError,
    DistFnoError,
    DTypeMismatchError,
    ExtensionMissingError,
    InfeasiblePartitionError,
    KernelError,
    MalformedHeaderError,
    NonFiniteLossError,
    SerializationError,
    TruncatedPayloadError,
    UnknownDTypeError,
    ReplicationError,
    ShapeMismatchError,
    UnknownLabelError,
)
from .fno import (
    ActivationKind,
    BlockCache,
    CommVolume,
    FnoConfig,
    FnoGrads,
    FnoParams,
    ForwardCache,
    clear_plans,
    decoder_forward,
    encoder_forward,
    fno_backward,
    fno_block_backward,
    fno_block_forward,
    fno_forward,
    init_params,
    predicted_block_volume,
    shard_params,
    slice_local,
)
from .partition import BlockRange, Partition, TransferBlock, block_decompose, range_intersection, repartition_plan
from .dtns import gather_params, load_checkpoint, save_checkpoint, serialized_size, tensor_from_bytes, tensor_read, tensor_to_bytes, tensor_write
from .graph import FwdBwdGraph
from .staging import InputStager
from .training import AdamState, adam_update, global_output_count, train_step
from .spectral import ModeSpec, fft_dims, ifft_dims, pad_modes, retained_extent, retained_indices, truncate_modes
from .tensor import (
    DATA_LABELS,
    DenseTensor,
    DimLabel,
    DType,
    bit_equal,
    einsum_channel_mix,
    einsum_spectral,
)

__version__ = "0.1.0"
