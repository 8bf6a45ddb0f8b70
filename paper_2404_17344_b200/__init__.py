"""B200-native NFFT fast summation for additive kernels (arXiv 2404.17344).

Drop-in for the hot path of the reference package ``addkern``: the feature
windows, the kernel setup and the matvec / derivative-matvec calls keep their
names and semantics, while the products run as hand-written sm_100a CUDA
kernels behind the C ABI in include/addkern_b200.h (libaddkern_b200.so).
There is no CPU compute path: without a CUDA device the compute calls raise.
"""

__version__ = "0.1.0"

from .dataset import (Dataset, ScalingFactor, from_arrays, minmax_to_quarter_box, prescale,
                      train_test_split, zscore_normalize)
from .kernels import KernelSpec, eval_kernel
from .windows import WindowSet, consec_windows, singleton_windows

__all__ = [
    "Dataset", "ScalingFactor", "KernelSpec", "WindowSet", "from_arrays", "zscore_normalize",
    "minmax_to_quarter_box", "prescale", "train_test_split", "eval_kernel", "consec_windows",
    "singleton_windows", "__version__",
]
