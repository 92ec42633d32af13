"""B200-native (sm_100a) Householder-product apply library for arXiv:1811.07624.

C ABI: include/hh.h, implemented by libhh.so (csrc/).  Python binding: .hh.
"""
from .hh import (HH_ALGO_AUTO, HH_ALGO_FUSED, HH_ALGO_WY, HH_SIDE_LEFT, HH_SIDE_RIGHT, algo,
                 debug_wy_project, hh_apply_signed, hh_get_algo, hh_knn, hh_set_algo,
                 hh_sym_apply_signed)
from .hh import HH_CALL_CONGRUENCE, HH_CALL_KNN, HH_CALL_SHF, hh_apply_qr, hh_congruence, hh_shf_cost  # noqa: F401
from .hh import (HH_CALL_APPLY, HH_CALL_APPLY_HOST, HH_CALL_MAHALANOBIS, HH_CALL_SYM, HH_F32,
                 HH_F64, HH_OP_N, HH_OP_T, HHError, hh_apply, hh_apply_host, hh_mahalanobis,
                 hh_sym_apply, hh_workspace_bytes, last_launch_info, lib, version)

__all__ = ["hh_apply", "hh_sym_apply", "hh_mahalanobis", "hh_apply_host", "hh_workspace_bytes",
           "HH_OP_N", "HH_OP_T", "HH_F32", "HH_F64", "HH_CALL_APPLY", "HH_CALL_SYM",
           "HH_CALL_MAHALANOBIS", "HH_CALL_APPLY_HOST", "HHError", "lib", "version",
           "last_launch_info", "HH_ALGO_AUTO", "HH_ALGO_FUSED", "HH_ALGO_WY", "algo",
           "hh_set_algo", "hh_get_algo", "debug_wy_project", "hh_apply_signed",
           "hh_sym_apply_signed", "HH_SIDE_LEFT", "HH_SIDE_RIGHT", "hh_knn", "HH_CALL_KNN",
           "hh_congruence", "HH_CALL_CONGRUENCE", "hh_apply_qr", "hh_shf_cost", "HH_CALL_SHF"]
