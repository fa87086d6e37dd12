"""B200 runtime for lowered *hyper* hash programs.

``program``  lowered-program records, the reference printer's text form, and
             an adapter for reference ``HirModule`` objects;
``lowering`` ``crypto.hash_batch`` -> per-GPU launch groups (partition +
             staging contract of ``lower_hyper_for``), fixed width and
             variable length (offsets re-based per shard);
``devices``  host + ``cuda`` device table (``detect_hardware``);
``executor`` ``execute`` / ``execute_batched`` on real GPUs;
``sweep``    ``Workload`` / ``run_point`` / ``sweep`` over GPU duty-ratio splits.
"""

from .devices import DeviceConfigError, DeviceSpec, DeviceTable, HOST_ID, detect_hardware, from_reference
from .executor import ExecError, ExecReport, execute, execute_batched
from .lowering import LoweringError, lower_hash_batch, lower_hash_batch_varlen
from .program import BufType, DigestLoop, Op, Program, ProgramError, VarDigestLoop, from_hir, parse
from .sweep import RunRecord, Workload, ratio_grid, records_to_csv, run_point, split_ratios, sweep, sweep_argmin

__all__ = ["DeviceConfigError", "DeviceSpec", "DeviceTable", "HOST_ID", "detect_hardware", "from_reference",
           "ExecError", "ExecReport", "execute", "execute_batched", "LoweringError", "lower_hash_batch",
           "lower_hash_batch_varlen", "VarDigestLoop",
           "BufType", "DigestLoop", "Op", "Program", "ProgramError", "from_hir", "parse", "RunRecord", "Workload",
           "run_point", "ratio_grid", "split_ratios", "sweep", "sweep_argmin", "records_to_csv"]
