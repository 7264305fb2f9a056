"""paper_1308_1536_b200 -- B200-native (sm_100a) drop-in for the hot path of
arXiv:1308.1536 (reference package `detseries`): arbitrary-precision,
unpivoted Gaussian elimination returning every leading principal minor and
the signed/normalized last-column minors for every leading size.

Public API mirrors the reference modules:
  scalars  : Precision, parse_scalar, format_scalar, agree_digits,
             canonical_bits, same_bits
  matrix   : MatrixBuffer
  elim     : eliminate, apply_pivot_to_row, minors_row_from_l,
             normalize_minors, laplace_residual, EliminationTrace,
             MinorRow, MinorSeries
  parexec  : par_eliminate, WorkerTopology, CommStats, pack_row, unpack_row
  genmat   : load_zeros, beta_matrix, power_matrix, synth_matrix, SpougeGamma
  errors   : the reference exception tree (+ DeviceUnavailable)
The elimination runs in libdetseries_b200.so (see include/detseries_b200.h);
importing the package does not touch the GPU.
"""

__version__ = "0.1.0"

from .errors import (CorruptPayload, DetseriesError, DeviceUnavailable, NormalizationUndefined,  # noqa: F401
                     ParseError, PrecisionMismatch, WorkerFailure, ZeroPivot)
from .scalars import (Precision, agree_digits, canonical_bits, format_scalar, parse_scalar,  # noqa: F401
                      same_bits)
from .matrix import MatrixBuffer  # noqa: F401
from .elim import (EliminationTrace, MinorRow, MinorSeries, apply_pivot_to_row, eliminate,  # noqa: F401
                   laplace_residual, minors_row_from_l, normalize_minors)
from .parexec import CommStats, WorkerTopology, pack_row, par_eliminate, unpack_row  # noqa: F401
from .genmat import SpougeGamma, beta_matrix, load_zeros, power_matrix, synth_matrix  # noqa: F401
from .output import write_dets, write_minors, write_results  # noqa: F401
