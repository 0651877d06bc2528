"""paper_2504_11681_b200 — B200-native (sm_100a) TurboFNO Fourier layer.

Drop-in for the reference package ``fnofuse``'s hot path (the 1D/2D
spectral-layer forward ``run_layer`` / ``run_fused`` / ``run_staged``, its
FFT and CGEMM APIs and the traffic ledger): same names, argument order,
shapes, truncation / zero-padding semantics and errors.  Compute runs in
hand-written CUDA kernels for sm_100a behind the C ABI ``include/turbofno.h``
(``libturbofno.so``); there is no CPU fallback.
"""

from .core import (COMPLEX_BYTES, COMPLEX_DTYPE, DEFAULT_TILES, FFT_BLOCK_BATCH, TALL_TILES,  # noqa: F401
                   WIDE_TILES, ConfigError, ConstraintViolation, FnoLayerConfig, FnofuseError,
                   ShapeMismatch, SpectralTensor, TileConfig, config_violations, max_rel_error,
                   random_spectral, tile_violations, validate_config)
from .fft import (FORWARD, INVERSE, FftPlan, InvalidKeep, InvalidLength, InvalidSrcLen,  # noqa: F401
                  LengthMismatch, OpCount, StrideOverlap, batched_execute, execute, execute_device,
                  full_op_count, plan)
from .cgemm import ComplexMatrix, GemmProblem, cgemm_device, gemm_kloop, gemm_tiled  # noqa: F401
from .pipeline import (ARRAY_NAMES, MODES, ConfigMismatch, FusedSchedule, ScheduleInvalid,  # noqa: F401
                       TrafficDelta, TrafficLedger, build_schedule, layer_flops, layer_op_stats,
                       PackedWeights, layer_schedule, model_ledger, prepare_weights, run_fused, run_layer,
                       run_layer_device, run_staged,
                       traffic_delta, workspace_bytes)

from .autograd import layer_backward, spectral_layer  # noqa: F401,E402  (backward pass, §8f row 4)
from .realfield import fno_block, real_layer  # noqa: F401,E402  (R2C/C2R layer, bypass + activation, §8f row 4)

__version__ = "0.1.0"
