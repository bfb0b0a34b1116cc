"""B200-native EDGC data-parallel hot path (arxiv 2511.10333).

Drop-in for the reference's public surface (pkg/src/edgc/__init__.py:15-85)
on the hot path: entropy estimation, entropy-to-rank model, window rank
scheduler, low-rank compress/decompress with error feedback, plus the
data-parallel bucket engine that replaces train_toy's per-worker loop.
Device work runs in libedgc_b200.so (hand-written sm_100a CUDA, ctypes C-ABI);
there is no CPU fallback.
"""

from .calibrate import calibrate_gpu, fit_comm_model, measure_compressor_gpu, write_comm_model
from .compressor import (CompressorState, LowRankFactors, compress, compressed_element_count, decompress,
                         set_rank)
from .controller import (CommModel, RankBounds, RankControllerState, RankDecision, adjust_rank_window,
                         align_stage_ranks, calibrate_comm_model, clamp_rank_step, compute_rank_bounds,
                         warmup_step)
from .entropy import (EntropyTracker, EntropyWindow, SamplerConfig, close_window, entropy_gaussian_plugin,
                      entropy_histogram, relative_change_rate, should_sample_iteration, subsample_entries)
from .errors import (CalibrationError, CompressionInfeasibleError, ConfigError, DegenerateInputError,
                     DivergenceError, EdgcError, TraceFormatError)
from .matrix_core import GradientMatrix, frobenius_norm, optimal_rank_r_error, pearson_correlation
from .trace import analyze_trace, read_trace_header, replay_trace, write_trace
from .rank_model import (GTable, MpSupport, build_g_table, estimate_g, g_table, invert_g, mp_cdf, mp_support,
                         rank_from_entropy, rank_from_sigma, sample_eigenvalues)

__version__ = "0.1.0"
