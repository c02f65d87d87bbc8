"""paper_2512_04556_b200: the Sparse Kernel Complex hot path on NVIDIA B200 (sm_100a).

A drop-in for the filtering, spatially varying filtering and kernel-fitting
API of the reference `sparsekern` package (arXiv 2512.04556): same names,
signatures and errors, with the arithmetic in hand-written CUDA kernels
(libskc.so, C ABI in include/skc.h).  `HAVE_CUDA` mirrors the reference's
`_fastpath.HAVE_NUMBA` switch; there is no CPU fallback.
"""

from ._native import NativeError, NativeUnavailable, release_scratch
from .engine import (
    EngineError,
    KernelComplex,
    SparseLayer,
    TruncationError,
    apply_complex,
    apply_complex_batch,
    apply_sparse_layer,
    auto_canvas,
    bilinear_sample,
    dense_convolve,
    psnr,
    required_canvas,
    sse,
    synthesize_ir,
    synthesize_ir_batch,
)
from .kernels import (
    DenseKernel,
    KernelError,
    KernelSpec,
    delta_kernel,
    disk_kernel,
    gaussian_kernel,
    generate_kernel,
    heart_kernel,
    load_kernel_image,
    polygon_kernel,
    read_image,
    ring_kernel,
    save_kernel_image,
    star_kernel,
    write_image,
)
from .optim import (
    AdamState,
    ConstraintConfig,
    FitResult,
    LossKind,
    OptimError,
    TrainConfig,
    adam_step,
    backward,
    backward_batch,
    fit,
    fit_batch,
    load_theta,
    loss,
    parse_layout,
    save_theta,
)
from .initializers import (
    InitStrategy,
    bbox_random_init,
    build_init,
    hybrid_init,
    radial_init,
    ss_init,
    support_rejection_sample,
)
from .baselines import PSTConfig, PSTResult, pst_fit
from .svfilter import (
    FilterBasis,
    FilterBasisGrid,
    build_basis,
    build_basis_grid,
    interp_weights,
    load_basis,
    save_basis,
    sv_filter,
    sv_filter_grid,
    sv_ground_truth,
    synthesize_filter,
)

__version__ = "0.2.0"


def __getattr__(name):
    # the reference's _fastpath.HAVE_NUMBA role; evaluated lazily so that
    # `import paper_2512_04556_b200` never loads libskc.so by itself
    if name == "HAVE_CUDA":
        from . import _native
        return _native.have_cuda()
    raise AttributeError(name)
