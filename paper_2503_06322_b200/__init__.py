"""B200-native MGARD reduction path of HPDR (arXiv 2503.06322).

Drop-in for the reference's ``hpdr.mgard`` / ``hpdr.huffman`` entry points; every stage
runs as hand-written sm_100a CUDA in ``libhpdr_b200.so`` (see include/hpdr_b200.h).
"""
from .context import Context, ContextCache, ContextKey
from .errors import (AllocationError, CorruptStreamError, DeviceError, FormatError, HpdrError,
                     StagingCapacityError, ValidationError)
from .hierarchy import Hierarchy, build_hierarchy
from .huffman import huffman_compress, huffman_decompress
from .mgard import (CoefficientSet, QuantizedSet, blob_info, compress, decompose, decompress, dequantize,
                    mgard_compress, mgard_decompress, quantize, recompose)
from .tensor import DTYPE_CODES, DTYPE_FROM_CODE, DType, TensorData
from .zfp import zfp_compress, zfp_decompress

__version__ = "0.1.0"

__all__ = [
    "AllocationError", "CoefficientSet", "Context", "ContextCache", "ContextKey", "CorruptStreamError", "DType",
    "DTYPE_CODES", "DTYPE_FROM_CODE", "DeviceError", "FormatError", "Hierarchy", "HpdrError", "QuantizedSet",
    "StagingCapacityError", "TensorData", "ValidationError", "blob_info", "build_hierarchy", "compress",
    "decompose", "decompress", "dequantize", "huffman_compress", "huffman_decompress", "mgard_compress",
    "mgard_decompress", "quantize", "recompose", "zfp_compress", "zfp_decompress",
]
