"""B200-native G-NetMon flow-analysis hot path (arXiv 1108.1785).

Flow-record batch + site registry in, per-site transfer-rate table and
sub-optimal-site flags out, computed by hand-written sm_100a kernels behind
the C-ABI in include/gnetmon.h. ``flowmon`` mirrors the reference C++ API.
"""
from . import flowmon  # noqa: F401  (loads lib/libgnetmon.so; fails loudly if absent)
from .flowmon import (AnalysisResult, ArchiveError, CatalogError, Cidr, ClassTallies, Engine, FilterParams,
                      FlowBatch, FlowClass, FlowRecords, GnmError, Group, LookupMode, RateStats,
                      SiteCatalog, SiteResult, SiteWarning, WarningState, aggregate,
                      aggregate_partitioned, evaluate_warnings, format_ipv4, parse_ipv4)

__all__ = [
    "AnalysisResult", "ArchiveError", "CatalogError", "Cidr", "ClassTallies", "Engine", "FilterParams",
    "FlowBatch", "FlowClass", "FlowRecords", "GnmError", "Group", "LookupMode", "RateStats", "SiteCatalog",
    "SiteResult", "SiteWarning", "WarningState", "aggregate", "aggregate_partitioned",
    "evaluate_warnings", "format_ipv4", "parse_ipv4",
]
