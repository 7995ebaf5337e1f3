"""B200-native incremental-TTS serving path (arXiv 2211.13939).

Instant Request Pooling + Module-wise Dynamic Batching behind the
reference's ``PipelineModules`` plugin boundary, with the encoder, the
chunked decoder and the chunk vocoder running as hand-written sm_100a
CUDA kernels reached through the C-ABI library ``libincrtts_b200.so``
(see ``include/incrtts_b200.h``).  Host modules mirror the reference
package ``incrtts`` name for name.
"""

from .audio import CrossfadeCurve, VocoderState, crossfade_curve, pcm16_decode, pcm16_encode, write_wav
from .domain import AudioChunk, ConfigError, MelChunk, PipelineConfig, load_config, validate_config
from .frontend import FrontendOutput, Lexicon, default_lexicon, g2p, load_lexicon, run_frontend
from .scheduler import (ChunkStream, CostModel, IterationReport, ModuleCost, PipelineModules,
                        PoolClosed, RequestCancelled, RequestFailed, RequestPool, SchedulerLoop,
                        latency_bounds, run_iteration, run_loop, write_iteration_log)

__version__ = "0.1.0"
