"""B200-native online stage of the method of polarized traces (arXiv 1410.5910).

The package is a drop-in for the reference's online GMRES solve
(``helmsweep.solver``): same public names, with the interface-operator
applies, the Gauss-Seidel sweeps and GMRES running as hand-written sm_100a
CUDA behind the C ABI of ``include/pt_b200.h`` (libpt_b200.so).

Modules:
  solver    reference-shaped API (gmres_solve, preconditioner_apply, ...)
  operator  DeviceOperator: one uploaded polarized operator (pt_handle)
  cache     PTC1 on-disk operator cache (offline results, reused across runs)
  capture   flatten a reference OfflineState into the upload tables
  _native   ctypes binding of libpt_b200.so
"""

__version__ = "0.1.0"

from .cache import read_case, write_case  # noqa: F401
