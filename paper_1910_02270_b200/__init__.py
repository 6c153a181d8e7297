"""B200-native LTFB hot path (arXiv 1910.02270): tournament training of the
JAG/ICF cycle-consistent surrogate on sm_100a.

The compute path is libltfb_gpu.so (csrc/, C ABI in include/ltfb_gpu.h);
this package is the Python mirror of the reference's trainer / model /
tournament API on top of that ABI.
"""
from ._lib import (CapacityError, ConfigError, ContractError, CudaError, DimensionError, Error,
                   IoError, NumericError, StoreCorruptError, LIB_PATH)
from .api import (AdamState, AutoencoderPretrainer, Comm, ae_batch_rows, pretrain_autoencoder, CycleGan, Dataset, SparseDataset, SynthDataset, BundleDataset, write_synth_bundles, synth_generate_device, synth_generate_ids, EpochRecord, EvalMetric, EvalRecord, HistorySegment,
                  Matching, ModalityDims, RoundRecord, RoundResult, StepRecord, SurrogateArch,
                  Trainer, TrainerConfig, TrainerRoundRecord, TransferRecord, device_count,
                  epoch_permutation, fnv1a64, hex64, incoming_wins, layer_widths, make_cyclegan,
                  mix_seed, pair_trainers, param_count, partition_dataset, reinit_gan_nets,
                  split_dataset, synth_generate, synthetic_dataset, tournament_round)

from .runner import (NcclRoundComm, RunConfig, RunHistory, RunResult, TorchRoundComm, TrainerSummary,
                     distributed_round, ensure_dataset, run_experiment, sharded_validation, run_experiment_rank, trainer_summary, warm_peer_links)
from .outputs import (config_from_json, config_hash, config_to_json, events_jsonl, load_model, save_model,
                      summary_csv, timings_csv, write_run_outputs)

__all__ = [n for n in dir() if not n.startswith("_")]
