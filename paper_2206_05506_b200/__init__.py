"""B200-native PN-correlation channel estimation (arXiv 2206.05506 hot path).

Front end mirroring the reference package `pnce` for the estimation path;
compute runs in libpnce_b200.so (sm_100a tcgen05/TMA kernels) via a C ABI.
"""

from .errors import *  # noqa: F401,F403
from .estimator import (CirEstimate, Correlator, WorkCounters, correlator_rows_for_plan,  # noqa: F401
                        process_frames, remove_cp)
from . import iqfile, operators, sweeps, synth  # noqa: F401
from .operators import (RowsCorrelator, batched_lag_rows, build_partial_circulant, correlate_rows,  # noqa: F401
                        estimate_batched, estimate_sequential, validate_batch_separation)
from .metrics import mae, mse  # noqa: F401
from .pilots import (BatchAssignment, BatchPlan, PilotConfig, PilotFrame, build_batch_plan,  # noqa: F401
                     build_pilot, cyclic_separation, max_batch, propagation_time, shift_for_transmitter)
from .pn import (PRIMITIVE_TAPS, LfsrSpec, PnSequence, circular_autocorrelation, circular_shift,  # noqa: F401
                 default_spec, generate_mseq, sequence_for_length)

__version__ = "0.1.0"
