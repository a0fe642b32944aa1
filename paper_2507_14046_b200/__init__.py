"""B200-native DIP-step engine for D²IP (arXiv 2507.14046).

Drop-in for the reference package's hot path (`pkg/src/d2ip/pipeline.py`
`_FrameOptimizer` and its drivers): the same Python API, with every
arithmetic step of a DIP iteration in hand-written sm_100a kernels behind the
C ABI of `include/d2ip_b200.h` (ctypes-bound in `_native.py`).
"""

from .errors import (  # noqa: F401
    DegenerateOperatorError,
    FormatError,
    NativeLibraryError,
    NumericalError,
    ReconstructionAborted,
)
from .forward import (  # noqa: F401
    ConductivitySequence,
    MaskedSensitivity,
    SensitivityMatrix,
    VoltageFrame,
    VoltageSequence,
    forward_project,
)
from .model import DeviceModel, build_model, extract_parameters, forward_volume, load_parameters  # noqa: F401
from .geometry import GridGeometry, cylinder_mask, devectorize, vectorize  # noqa: F401
from .priornet import (  # noqa: F401
    NetworkConfig,
    NoiseInput,
    ParameterState,
    ResUNetConfig,
    count_parameters,
    init_parameters,
    load_checkpoint,
    sample_noise_input,
    save_checkpoint,
)
from .regularizers import FrameHistory, TVWeights, decay_weight, spatial_tv, temporal_tv, tv4d  # noqa: F401
from .sensitivity import (  # noqa: F401
    assemble_masked_device,
    assemble_sensitivity,
    load_matrix,
    load_matrix_device,
    load_voltages,
    normalize_sensitivity,
    save_matrix,
    save_voltages,
)
from .pipeline import (  # noqa: F401
    LossTrace,
    BatchedSequenceResult,
    ReconstructionResult,
    RunConfig,
    ablation_mode,
    derived_seeds,
    loss,
    predict_measurements,
    reconstruct_frame,
    joint_upws_pretrain,
    reconstruct_sequence,
    reconstruct_sequence_joint,
    reconstruct_sequences_batched,
    upws_pretrain,
)

__version__ = "0.1.0"
