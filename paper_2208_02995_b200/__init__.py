"""B200-native restricted-PCG energy minimisation of an AMG prolongation
(arXiv 2208.02995): C-ABI library libemin.so (csrc/, include/emin.h) and its
thin Python binding.  Never imports ``oracle`` (test infrastructure)."""
from .emin import (Emin, EminError, emin_destroy, emin_energy, emin_get_P, emin_iterate,  # noqa: F401
                   emin_get_layout,
                   emin_kernel_times, emin_report, emin_reset, emin_set_profiling, emin_setup,
                   load_library, LIB_PATH, EXPORTED)
from .build import build  # noqa: F401
