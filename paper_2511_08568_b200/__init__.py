"""B200-native RecMG hot path (arxiv 2511.08568), drop-in for the reference
``embcache`` replay / model / buffer-simulator API.

The compute runs in hand-written sm_100a kernels (csrc/) behind the C ABI
in include/recmg.h, loaded from the in-tree librecmg.so; there is no CPU
fallback on this path.
"""
from .checkpoint import load_checkpoint, load_checkpoint_shard, save_checkpoint, vocabulary_hash
from .cache_sim import (CacheConfig, Policy, SimResult, brute_force_optimal, simulate,
                        simulate_optgen, sweep, write_sweep_csv)
from .errors import (CheckpointError, EmbcacheError, InvalidConfigError,
                     MissingArtifactError, NumericalError, OutOfVocabularyError,
                     TraceParseError, TraceValidationError, VocabularyMismatchError)
from .labeler import (LABEL_CAPACITY_FRACTION, LabeledDataset, caching_label_array,
                      label_caching, label_prefetch, prefetch_target_array, read_dataset,
                      split_dataset, write_dataset)
from .model import (CACHING, PREFETCH, DeviceModel, ModelParameters, batch_arrays,
                    decode_indices, device_model, forward_caching, forward_caching_batch,
                    forward_prefetch, forward_prefetch_batch, init_params,
                    invalidate_device_models, normalize_gids)
from .runtime import (EVICTION_SPEED, BreakdownReport, BufferConfig, PriorityBuffer,
                      correctness_vs_window, coverage, gpu_buffer_populate, load_embeddings,
                      optgen_miss_oracle, replay, replay_policy_only, write_breakdown_csv)
from .trace import (EmbeddingIndex, SequenceSample, Trace, TraceGenConfig, chunk,
                    TraceStream, generate_trace, generate_trace_streamed, index_of_global,
                    make_index, num_chunks, read_trace, read_trace_binary, table_offsets,
                    trace_from_gids, write_trace, write_trace_binary)

__version__ = "0.1.0"
