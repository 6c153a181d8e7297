"""ctypes binding of include/ltfb_gpu.h (libltfb_gpu.so, built in-tree).

There is no fallback: if the CUDA library is missing the import fails with
instructions to build it (python -c "import __graft_entry__ as g; g.build()").
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LTFB_LIB_PATH") or os.path.join(PKG, "_build", "libltfb_gpu.so")  # override: A/B runs


class Error(RuntimeError):
    """ltfb::Error (core/error.hpp:11-14)."""


class DimensionError(Error):
    pass


class ContractError(Error):
    pass


class NumericError(Error):
    pass


class IoError(Error):
    pass


class CapacityError(Error):
    pass


class StoreCorruptError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    pass


_CODES = {1: DimensionError, 2: ContractError, 3: NumericError, 4: IoError, 5: CapacityError,
          6: StoreCorruptError, 7: ConfigError, 8: CudaError, 9: Error}

NET_ENC, NET_DEC, NET_FWD, NET_INV, NET_DISC = range(5)
SLICE_TOURNAMENT, SLICE_VALIDATION = 0, 1


class Dims(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("input_dim", "latent_dim", "scalar_dim", "image_views",
                                          "image_channels", "image_h", "image_w")]


class Arch(C.Structure):
    _fields_ = ([(n, C.c_uint32 * 8) for n in ("enc_hidden", "dec_hidden", "fwd_hidden",
                                               "inv_hidden", "disc_hidden")]
                + [(n, C.c_uint32) for n in ("n_enc_hidden", "n_dec_hidden", "n_fwd_hidden",
                                             "n_inv_hidden", "n_disc_hidden")]
                + [("hidden_act", C.c_int32), ("hidden_slope", C.c_double),
                   ("lambda_adv", C.c_double), ("lambda_cyc", C.c_double), ("lr", C.c_double),
                   ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)])


class TrainerConfigC(C.Structure):
    _fields_ = [("trainer_id", C.c_int32), ("device", C.c_int32), ("n_shards", C.c_int32),
                ("numeric_abort_threshold", C.c_int32), ("batch_size", C.c_uint64),
                ("seed", C.c_uint64), ("w_f", C.c_double), ("w_i", C.c_double),
                ("lr_fwd", C.c_double), ("lr_inv", C.c_double), ("lr_disc", C.c_double),
                ("wide_kernel", C.c_int32), ("post_kernel", C.c_int32)]


class StepRecordC(C.Structure):
    _fields_ = [("step", C.c_uint64), ("epoch", C.c_uint32), ("skipped", C.c_uint32),
                ("d_loss", C.c_double), ("g_total", C.c_double), ("g_fwd", C.c_double),
                ("g_adv", C.c_double), ("g_cyc", C.c_double)]


class EpochRecordC(C.Structure):
    _fields_ = [("epoch", C.c_uint32), ("partial", C.c_uint32), ("steps", C.c_uint64),
                ("samples_shuffled", C.c_uint64), ("seconds", C.c_double)]


class EvalMetricC(C.Structure):
    _fields_ = [("forward_mae", C.c_double), ("inverse_mae", C.c_double), ("combined", C.c_double)]


# every symbol include/ltfb_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "ltfb_last_error", "ltfb_abi_version", "ltfb_device_count", "ltfb_arch_defaults",
    "ltfb_trainer_create", "ltfb_trainer_destroy", "ltfb_trainer_param_count",
    "ltfb_trainer_set_params", "ltfb_trainer_get_params", "ltfb_trainer_set_adam",
    "ltfb_trainer_get_adam", "ltfb_trainer_load_store", "ltfb_trainer_set_slice",
    "ltfb_trainer_generate_store", "ltfb_trainer_generate_slice", "ltfb_synth_generate_device",
    "ltfb_dataset_open", "ltfb_dataset_destroy", "ltfb_dataset_info", "ltfb_dataset_file_of", "ltfb_dataset_read",
    "ltfb_write_synth_bundles",
    "ltfb_trainer_train_steps", "ltfb_trainer_step", "ltfb_trainer_take_epochs",
    "ltfb_trainer_flush_epoch", "ltfb_trainer_evaluate", "ltfb_trainer_generator_floats",
    "ltfb_trainer_get_generator", "ltfb_trainer_set_incoming", "ltfb_trainer_copy_incoming",
    "ltfb_trainer_tournament_decide", "ltfb_trainer_adopt", "ltfb_trainer_train_steps_host",
    "ltfb_trainer_timer_start", "ltfb_trainer_timer_stop", "ltfb_trainer_kernel_timing",
    "ltfb_trainer_kernel_time", "ltfb_trainer_wide_info", "ltfb_trainer_wide_tile", "ltfb_trainer_eval_info", "ltfb_trainer_ae_info", "ltfb_trainer_stream_info", "ltfb_trainer_stream_profile", "ltfb_trainer_launch_count",
    "ltfb_nccl_available", "ltfb_synth_generate_ids", "ltfb_selftest_tcgen05",
    "ltfb_nccl_unique_id", "ltfb_comm_create", "ltfb_comm_destroy", "ltfb_trainer_exchange",
    "ltfb_trainer_broadcast", "ltfb_mix_seed", "ltfb_fnv1a64", "ltfb_pair_trainers",
    "ltfb_partition_dataset", "ltfb_split_dataset", "ltfb_epoch_permutation",
    "ltfb_incoming_wins", "ltfb_synth_generate", "ltfb_init_params", "ltfb_net_param_count",
    "ltfb_trainer_synchronize", "ltfb_trainer_prepare_graphs", "ltfb_trainer_load_ae_source", "ltfb_trainer_ae_step", "ltfb_ae_batch_rows",
    "ltfb_adam_step", "ltfb_trainer_ae_alloc_source", "ltfb_trainer_ae_fill_from_store",
    "ltfb_trainer_ae_allgather",
)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 CUDA library has not been built. Run "
            "`python -c \"import __graft_entry__ as g; g.build()\"` from the repo root.")
    return C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)


lib = _load()
P = C.c_void_p
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


lib.ltfb_last_error.restype = C.c_char_p
_sig("ltfb_abi_version", C.c_int)
_sig("ltfb_device_count", C.c_int, C.POINTER(C.c_int))
_sig("ltfb_arch_defaults", None, C.POINTER(Arch))
_sig("ltfb_trainer_create", C.c_int, C.POINTER(Dims), C.POINTER(Arch), C.POINTER(TrainerConfigC),
     C.POINTER(P))
_sig("ltfb_trainer_destroy", C.c_int, P)
_sig("ltfb_trainer_param_count", C.c_int, P, C.c_int, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_set_params", C.c_int, P, C.c_int, f32p, C.c_uint64)
_sig("ltfb_trainer_get_params", C.c_int, P, C.c_int, f32p, C.c_uint64)
_sig("ltfb_trainer_set_adam", C.c_int, P, C.c_int, P, P, C.c_uint64)
_sig("ltfb_trainer_get_adam", C.c_int, P, C.c_int, P, P, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_load_store", C.c_int, P, u32p, C.c_uint64, f32p, f32p, P)
_sig("ltfb_trainer_set_slice", C.c_int, P, C.c_int, f32p, f32p, C.c_uint64)
_sig("ltfb_trainer_generate_store", C.c_int, P, u32p, C.c_uint64, P, C.c_uint64, C.c_double, C.c_uint64,
     C.c_uint64)
_sig("ltfb_trainer_generate_slice", C.c_int, P, C.c_int, u32p, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
     C.c_uint64)
_sig("ltfb_trainer_train_steps", C.c_int, P, C.c_uint64, C.POINTER(StepRecordC), C.POINTER(C.c_uint64))
_sig("ltfb_trainer_step", C.c_int, P, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_take_epochs", C.c_int, P, C.POINTER(EpochRecordC), C.c_uint64, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_flush_epoch", C.c_int, P)
_sig("ltfb_trainer_evaluate", C.c_int, P, C.c_int, P, P, C.c_double, C.c_double, C.POINTER(EvalMetricC))
_sig("ltfb_trainer_generator_floats", C.c_int, P, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_get_generator", C.c_int, P, f32p, C.c_uint64)
_sig("ltfb_trainer_set_incoming", C.c_int, P, f32p, f32p)
_sig("ltfb_trainer_copy_incoming", C.c_int, P, P)
_sig("ltfb_trainer_tournament_decide", C.c_int, P, C.POINTER(EvalMetricC), C.POINTER(EvalMetricC),
     C.POINTER(C.c_int32))
_sig("ltfb_trainer_adopt", C.c_int, P, f32p, f32p)
_sig("ltfb_trainer_train_steps_host", C.c_int, P, C.c_uint64, P, P, C.POINTER(StepRecordC),
     C.POINTER(C.c_uint64))
_sig("ltfb_trainer_timer_start", C.c_int, P)
_sig("ltfb_trainer_timer_stop", C.c_int, P, C.POINTER(C.c_double))
_sig("ltfb_trainer_kernel_timing", C.c_int, P, C.c_int)
_sig("ltfb_trainer_kernel_time", C.c_int, P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_uint64))
_sig("ltfb_trainer_wide_info", C.c_int, P, C.POINTER(C.c_int32), C.POINTER(C.c_int32))
_sig("ltfb_trainer_wide_tile", C.c_int, P, C.POINTER(C.c_int32))
_sig("ltfb_trainer_eval_info", C.c_int, P, C.c_int, C.POINTER(C.c_int32))
_sig("ltfb_trainer_ae_info", C.c_int, P, C.c_int32, C.POINTER(C.c_int32))
_sig("ltfb_trainer_stream_info", C.c_int, P, C.POINTER(C.c_int32))
_sig("ltfb_trainer_stream_profile", C.c_int, P, C.c_int, C.POINTER(C.c_double), C.c_int)
_sig("ltfb_trainer_launch_count", C.c_int, P, C.POINTER(C.c_uint64))
_sig("ltfb_synth_generate_ids", C.c_int, C.POINTER(Dims), C.c_uint64, C.c_double, u32p, C.c_uint64,
     C.c_uint64, C.c_uint64, f32p, f32p, C.c_int)
_sig("ltfb_nccl_available", C.c_int)
_sig("ltfb_selftest_tcgen05", C.c_int, f32p, f32p, f32p, f32p, f32p, f32p, f32p, f32p)
_sig("ltfb_trainer_ae_alloc_source", C.c_int, P, C.c_uint64)
_sig("ltfb_trainer_ae_fill_from_store", C.c_int, P, u32p, C.c_uint64, C.c_uint64)
_sig("ltfb_trainer_ae_allgather", C.c_int, P, P, C.c_uint64)
_sig("ltfb_adam_step", C.c_int, f32p, f32p, f32p, f32p, C.c_uint64, C.POINTER(C.c_uint64), C.c_double,
     C.c_double, C.c_double, C.c_double, C.c_int)
_sig("ltfb_nccl_unique_id", C.c_int, C.c_char_p)
_sig("ltfb_comm_create", C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(P))
_sig("ltfb_comm_destroy", C.c_int, P)
_sig("ltfb_trainer_exchange", C.c_int, P, P, C.c_int)
_sig("ltfb_trainer_broadcast", C.c_int, P, P, C.c_int, C.c_int)
_sig("ltfb_mix_seed", C.c_uint64, u64p, C.c_int)
_sig("ltfb_fnv1a64", C.c_uint64, C.c_void_p, C.c_uint64)
_sig("ltfb_pair_trainers", C.c_int, C.c_int, C.c_int, C.c_uint64, i32p, C.POINTER(C.c_int32),
     C.POINTER(C.c_int32))
_sig("ltfb_partition_dataset", C.c_int, u32p, C.c_uint64, C.c_int, C.c_uint64, u32p, u32p)
_sig("ltfb_split_dataset", C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int,
     u32p, C.POINTER(C.c_uint64), u32p, u32p, u32p, u32p)
_sig("ltfb_epoch_permutation", C.c_int, u32p, C.c_uint64, C.c_uint32, C.c_uint64, u32p)
_sig("ltfb_incoming_wins", C.c_int, C.c_double, C.c_double)
_sig("ltfb_synth_generate", C.c_int, C.POINTER(Dims), C.c_uint64, C.c_double, C.c_uint64, C.c_uint64,
     C.c_uint64, C.c_uint64, f32p, f32p, C.c_int)
_sig("ltfb_synth_generate_device", C.c_int, C.POINTER(Dims), C.c_uint64, C.c_double, P, C.c_uint64,
     C.c_uint64, C.c_uint64, C.c_uint64, P, P, C.c_uint64, C.c_int)
_sig("ltfb_dataset_open", C.c_int, C.c_char_p, C.POINTER(P))
_sig("ltfb_dataset_destroy", C.c_int, P)
_sig("ltfb_dataset_info", C.c_int, P, C.POINTER(Dims), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
_sig("ltfb_dataset_file_of", C.c_int, P, u32p, C.c_uint64, u32p)
_sig("ltfb_dataset_read", C.c_int, P, u32p, C.c_uint64, f32p, f32p, C.POINTER(C.c_uint64))
_sig("ltfb_write_synth_bundles", C.c_int, C.c_char_p, C.POINTER(Dims), C.c_uint64, C.c_double, C.c_uint64,
     C.c_uint64, C.c_uint32, C.c_int)
_sig("ltfb_init_params", C.c_int, C.POINTER(Dims), C.POINTER(Arch), C.c_uint64, C.c_int, f32p, C.c_uint64)
_sig("ltfb_net_param_count", C.c_int, C.POINTER(Dims), C.POINTER(Arch), C.c_int, C.POINTER(C.c_uint64))
_sig("ltfb_trainer_synchronize", C.c_int, P)
_sig("ltfb_trainer_prepare_graphs", C.c_int, P)
_sig("ltfb_trainer_load_ae_source", C.c_int, P, f32p, C.c_uint64)
_sig("ltfb_trainer_ae_step", C.c_int, P, u32p, C.c_uint64, C.POINTER(C.c_double))
_sig("ltfb_ae_batch_rows", C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p)


def check(rc: int):
    if rc != 0:
        msg = lib.ltfb_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
