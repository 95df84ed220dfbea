"""B200-native tensor-parallel selective-SSM (Mamba) mixer, arXiv 2602.21144.

The compute path is libssmtp.so (C ABI in include/ssm_tp.h, CUDA kernels for
sm_100a under csrc/).  This package is the thin Python binding (argument
marshalling, device memory and streams via PyTorch) plus the layer stack used by
bench.py.  Importing it fails loudly if the CUDA library has not been built.
"""
from ._lib import SSMError, SSM_AR2_EXTERNAL, SSM_AR2_FP32, SSM_AR2_INT8  # noqa: F401
from .mixer import LayerWeights, State, TPMixer, channel_range  # noqa: F401
