"""paper_2104_02621_b200 -- B200-native capsule convolution (arXiv 2104.02621).

The compute lives in libcapsconv.so (csrc/, C ABI in include/capsconv.h);
this package is the thin Python binding (capsconv.py) and the data-parallel
stack driver (stack.py).
"""
from .capsconv import (  # noqa: F401
    CapsConvError,
    CapsConvFunction,
    OP_BWD_DATA,
    OP_BWD_KERNEL,
    OP_FWD,
    PATH_AUTO,
    PATH_MMA,
    LAYOUT_NATURAL,
    LAYOUT_ROWS,
    PATH_SIMT,
    bwd_data,
    bwd_data_slices,
    bwd_kernel,
    bwd_kernel_slices,
    caps_conv2d,
    fwd,
    fwd_slices,
    launch_count,
    load_library,
    output_dims,
    select_path,
    set_path_override,
    version,
    workspace_bytes,
)
