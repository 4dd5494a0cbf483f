"""B200-native compressed tensor-parallel all-reduce (arXiv 2411.09510).

Drop-in for the reference package ``mxcomm`` on its hot path: the block
codec (formats / codec names re-exported unchanged) and the compressed
collective, computed by hand-written sm_100a kernels behind the C ABI of
``include/mxb200.h`` (``libmxb200.so``).  See DESIGN.md.
"""

from .errors import (BadMagic, MalformedCode, MalformedHeader, MinimumDegreeTwo, MxcommError,
                     NativeUnavailable, NonFiniteInput, ResultMismatch, ShapeMismatch,
                     TransportFailure, TruncatedStream, UnknownScheme, UnsupportedVersion)
from .formats import (ELEMENT_CODES, ELEMENT_FORMATS, EXTENSION_FORMATS, SCALE_CODES,
                      SCALE_FORMATS, ElementFormat, FormatKind, ScaleFormat, SchemeDescriptor,
                      ValueGrid, effective_bits, element_format, emax, enumerate_grid,
                      parse_scheme, scale_format)
from .codec import (CompressedTensor, DeviceCompressedTensor, block_error_bound,
                    compress_tensor, compress_tensor_device, decompress_tensor,
                    decompress_tensor_device, dequantize_block, deserialize, deserialize_device,
                    header_nbytes, pack_header, quantize_block, serialize, serialize_device,
                    serialized_nbytes, unpack_header)

from .baselines import (ChannelIntPacket, TopKPacket, channelwise_int_compress,
                        channelwise_int_decompress, topk_compress, topk_decompress)
from .errors import CompressionFactorTooHigh
from .tp import (ReductionReport, TPConfig, parallelism_sweep, shard_rowwise,
                 simulate_reduction)
from .netbench import (BenchResult, LinkModel, calibrate_codec_throughput, predict_comm_time,
                       predicted_speedup, run_allgather_bench)
from .search import (DeviceReductionEvaluator, make_activation_evaluator,
                     make_simulation_evaluator)
from .collective import (CompressedAllReduce, FusedLinearAllReduce, HostPipeline, LocalThreadGroup,
                         SimulatedAllReduce, SymmetricAllReduce, compressed_all_reduce)

__version__ = "0.1.0"
