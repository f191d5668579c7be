"""B200-native incremental RTEC engine (drop-in for the streamgnn hot path).

Public surface mirrors the reference (`streamgnn.graph`, `streamgnn.models`,
the SPEC engine API): see DESIGN.md.  All compute runs in librtec.so
(hand-written sm_100a CUDA) through the C ABI in include/rtec.h.
"""

from .errors import (  # noqa: F401
    ConfigError, InvalidVertex, NativeError, NumericError, ShapeError, SingularContext, StaleState, StreamGNNError,
    UnsupportedModel,
)
from .graph import (  # noqa: F401
    ApplyResult, DegreeDelta, DynamicGraph, EdgeUpdate, UpdateOp, coalesce_batch, invert_batch, read_stream,
    write_stream,
)
from .models import MODELS, Bundle, LayerWeights, from_reference, make_bundle  # noqa: F401
from .engine import (  # noqa: F401
    Metrics, RTECEngine, RunResult, forward_layer_reference, layer_embeddings, redundancy, reference_embeddings,
)

from .formats import (  # noqa: F401
    load_checkpoint, load_sharded_checkpoint, load_weights, read_tensor, save_checkpoint, save_sharded_checkpoint,
    save_weights, write_tensor,
)

__version__ = "0.1.0"
