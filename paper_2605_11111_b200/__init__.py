"""B200-native ShardTensor domain-parallel hot path (arxiv/paper_2605_11111).

Drop-in for the reference's operator API (`domainpar`): ShardTensor with
uneven per-rank shard shapes, Shard/Replicate placements, scatter_global /
full_tensor / redistribute, the dispatch table ("conv" -> halo_conv,
"ring_attention" -> ring_attention), and the mesh collectives — with device
tensors, sm_100a kernels behind a C ABI (libdpb200.so) and NCCL between
processes.  See DESIGN.md.
"""

from . import layers as _layers  # registers add/mul/scale/linear/softmax/layer_norm  # noqa: F401
from . import ops as _ops  # registers the default handlers  # noqa: F401
from .dispatch import (DEFAULT_TABLE, DENSE_REFERENCE, LEVELS, DispatchTable, OpKey,
                       TraceRecord, dispatch_operation, fallback_dispatch, promote_result,
                       register_dense_reference, register_handler, trace_lines)
from .errors import (CollectiveError, DegenerateInputError, DeviceError, DimensionError,
                     DomainParError, FitError, HaloError, IntegrityError, MeshError,
                     MetadataError, ShapeError, UnsupportedConfigError,
                     UnsupportedOperationError)
from .mesh import (AxisGroup, DeviceMesh, RankContext, all_gather_varlen, all_reduce, barrier,
                   halo_exchange, init_mesh, ring_shift, spawn_mesh)
from .ops import (AttnTape, ConvTape, HaloConv2, RingAttention, RingSoftmaxState, dense_conv,
                  halo_conv, halo_conv_autograd, halo_conv_backward, halo_conv_forward,
                  ring_attention, ring_attention_autograd, ring_attention_backward,
                  ring_attention_forward, sdpa_dense)
from .layers import (ELEMENTWISE_OPS, ActivationLedger, VitConfig, ddp_allreduce_grads,
                     dense_elementwise, dense_layer_norm, dense_linear, dense_matmul,
                     dense_softmax, image_to_sequence, make_vit_weights, sharded_elementwise,
                     sharded_layer_norm, sharded_linear, sharded_softmax, vit_block_pipeline,
                     vit_block_pipeline_dense)
from .plan import conv_output_extent, halo_conv_plan, owned_output_range
from .sharding import (Placement, Replicate, Shard, ShardTensor, default_chunk, full_tensor,
                       redistribute, replicated, scatter_global)

conv = dense_conv
__version__ = "0.1.0"
