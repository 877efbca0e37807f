# semopt/b200.py -- reference-side binding of libsemb200.so (include/sem1d.h).
#
# This is the file a semopt maintainer adds to the STOCK reference package: a SemOperator
# subclass whose three apply methods call the C ABI.  The reference's own integrate / sweep /
# AssimilationProblem / minimize then run unchanged on top of it.  It is
# executed against the unmodified reference installed in baseline/_ref by
# tests/test_gpu_dropin.py.  SEMB200_LIB names the library (default: the in-tree build).
import ctypes
import os

import numpy as np
import torch

from semopt.errors import NumericFailure, ValidationError
from semopt.ops import SemOperator

_LIB = os.environ.get("SEMB200_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "paper_1806_01422_b200", "libsemb200.so"))
_lib = ctypes.CDLL(_LIB)
vp, i64 = ctypes.c_void_p, ctypes.c_int64
_lib.sem1d_plan_create.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                   vp, vp, vp, vp, i64, ctypes.POINTER(vp)]
_lib.sem1d_plan_destroy.argtypes = [vp]
for name in ("sem1d_rhs",):
    getattr(_lib, name).argtypes = [vp, vp, vp, vp, vp]
for name in ("sem1d_jac", "sem1d_jact"):
    getattr(_lib, name).argtypes = [vp, vp, vp, vp, vp, vp]
_lib.sem1d_last_error.restype = ctypes.c_char_p


class B200SemOperator(SemOperator):
    """SemOperator whose applies run on the B200 (1D Burgers only)."""

    def __init__(self, grid, coef):
        super().__init__(grid, coef)                      # ops.py:91-124 constants
        ax, N = grid.axes[0], grid.axes[0].degree
        m = grid.mass_scalar                              # grid.py:128-131, assembled
        # per-position patterns (sem1d.h): [0] interface, [1..N-1] interior, [N], [N+1] ends
        mass = np.empty(N + 2)
        mass[1:N] = m[1:N]                                # interior nodes of element 0
        mass[0] = m[N % m.size]                           # node N: an interface (wraps if E = 1)
        mass[N], mass[N + 1] = m[0], m[-1]                # Dirichlet end nodes
        self._pat = (np.ascontiguousarray(mass), np.ascontiguousarray(1.0 / mass))
        self._plan = vp()
        rc = _lib.sem1d_plan_create(ax.elements, N, ax.bc == "periodic", coef.nu,
                                    self._kmat[0].ctypes.data, self._dw[0].ctypes.data,
                                    self._pat[0].ctypes.data, self._pat[1].ctypes.data,
                                    1, ctypes.byref(self._plan))
        if rc:
            raise ValidationError(_lib.sem1d_last_error().decode())
        self._flag = torch.zeros(1, dtype=torch.int32, device="cuda")

    def __del__(self):
        if getattr(self, "_plan", None) is not None and self._plan.value:
            _lib.sem1d_plan_destroy(self._plan)
            self._plan = None

    def _call(self, fn, names, *arrays):
        # ops.py:216-224 shape check; inputs through pinned buffers (torch's caching host
        # allocator), so the host->device copies run at DMA speed, not through pageable staging
        dev = [torch.from_numpy(np.ascontiguousarray(self._check(a, n))).pin_memory().cuda(non_blocking=True)
               for a, n in zip(arrays, names)]
        out = torch.empty_like(dev[0])
        fn(self._plan, *[d.data_ptr() for d in dev], out.data_ptr(), self._flag.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
        if int(self._flag.item()):                        # ops.py:222-223 semantics
            self._flag.zero_()
            raise NumericFailure(f"{names[0]} contains NaN/Inf")
        host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)   # a new array per call
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host.numpy()

    def _check(self, u, name):                            # shape only; NaN goes to the flag
        u = np.asarray(u, dtype=float)
        if u.shape != (self.grid.nglobal,):
            raise ValidationError(f"{name} has shape {u.shape}, expected ({self.grid.nglobal},)")
        return u

    def apply_rhs(self, u):
        self.counters["rhs"] += 1
        return self._call(_lib.sem1d_rhs, ("state",), u)

    def apply_jacobian(self, u, w):
        self.counters["jac"] += 1
        return self._call(_lib.sem1d_jac, ("state", "tangent"), u, w)

    def apply_jacobian_transpose(self, u, z):
        self.counters["jact"] += 1
        return self._call(_lib.sem1d_jact, ("state", "cotangent"), u, z)
