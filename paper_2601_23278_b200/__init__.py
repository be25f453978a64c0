"""B200-native (sm_100a) FOCUS block-diffusion decode step: C-ABI libfocus.so + thin binding.

Layout:
  csrc/        CUDA kernels + host orchestration behind include/focus.h (built by build.py)
  focus.py     ctypes binding (same names as the C ABI; argument marshalling only)
  runner.py    request driver used by bench.py, __graft_entry__.smoke() and the GPU tests
"""
from .focus import FocusContext, FocusError, make_config  # noqa: F401
