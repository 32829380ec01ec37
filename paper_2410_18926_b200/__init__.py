"""B200-native LoRANN query engine (arXiv 2410.18926), drop-in for ``rrann.query_batch``.

Public API (mirrors pkg/src/rrann/__init__.py:11-21 for the query path):
``query``, ``query_batch``, ``QueryParams``, ``QueryResult``, the error
classes, plus ``DeviceIndex`` (device-resident index) and its
``search_device`` entry used for throughput measurement.
"""

from .errors import BuildError, DataError, FormatError, ParameterError, RrannError, ShapeError
from .device_index import DeviceIndex, last_launch_count, version
from .ground_truth import brute_force_knn, ground_truth_device
from .search import QueryParams, QueryResult, device_index_for, install, query, query_batch

__all__ = [
    "BuildError", "DataError", "DeviceIndex", "FormatError", "ParameterError", "QueryParams",
    "QueryResult", "brute_force_knn", "ground_truth_device", "RrannError", "ShapeError", "device_index_for", "install", "last_launch_count",
    "query", "query_batch", "version",
]

__version__ = "0.1.0"
