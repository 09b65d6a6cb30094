"""Decoder-layer bookkeeping kept on the host.

The decoder layer itself (layers.py:66-119 in the reference) runs on the
GPU inside libgr4ad; this module keeps the reference's instrumentation API.
"""

import threading

LN_EPS = 1e-5  # layers.py:15


class LayerCallCounter:
    """Same contract as ``adrec.model.layers.LayerCallCounter``
    (layers.py:18-35): decoder-layer row applications, KV builds and the
    largest cross-attention KV footprint in floats.  Thread-safe.  The GPU
    decode updates it from the closed forms instead of
    doing the reference's padded work."""

    def __init__(self):
        self._lock = threading.Lock()
        self.layer_calls = 0
        self.kv_builds = 0
        self.kv_floats = 0

    def add_layer_calls(self, rows):
        with self._lock:
            self.layer_calls += int(rows)

    def add_kv_build(self, builds, floats):
        with self._lock:
            self.kv_builds += int(builds)
            self.kv_floats = max(self.kv_floats, int(floats))
