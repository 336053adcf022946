"""CPU dry-run backend for bench.py (TEST INFRASTRUCTURE; selected with
PE_BENCH_BACKEND=tests.bench_cpu_backend:CpuBackend).

It lets the multi-process logic of `bench.py --gpus N` (torchrun re-exec, interval
sharding, the all-gather per iteration, max-over-ranks timing, the JSON line) run under
gloo on CPU.  The device context is the CPU oracle stand-in of tests/test_sharded.py; no
number from such a run is a measurement.
"""

import time

import numpy as np
import torch

from oracle import pe_oracle as po
from tests.test_sharded import OracleOps


class _Event:
    def record(self):
        self.t = time.perf_counter()

    def elapsed_time(self, other):
        return (other.t - self.t) * 1e3


class _NoClock:
    result = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class OracleContext:
    """The PeContext methods bench.py's sharded path calls, on the CPU oracle (member 0)."""

    def __init__(self, systems, loads, J, T, N, alpha):
        s = systems[0]
        ld = loads[0]
        self.osys = po.OSystem(s.M11, s.A11, s.M12, s.A12, s.M22, s.A22, ld.f1, ld.f2)
        self.J, self.T, self.N, self.alpha = J, T, N, alpha
        self.ops = {}
        self.d = s.d1 + s.d2
        self.launches = 0

    def _ops(self, kind):
        if kind not in self.ops:
            self.ops[kind] = OracleOps(self.osys, self.T, self.N, self.J, kind, self.alpha)
        return self.ops[kind]

    def prepare_coarse(self, dt):
        pass

    def prepare_sequential(self, dt):
        pass

    def prepare_allatonce(self, dt, alpha, tol, max_iter):
        pass

    def modal_level(self):
        return 0

    def to_dev(self, x):
        return torch.as_tensor(np.array(x, dtype=np.float64))

    def fine_sequential(self, X):
        self.launches += 1
        return self._ops("sequential").fine(X)[0]

    def fine_allatonce(self, X, record=True):
        self.launches += 1
        Y, sw = self._ops("all-at-once").fine(X)
        return Y, sw[None], None, None

    def coarse_correct(self, N, X_old, F_hat, G_cache, X_new, diff=None, active=None):
        self.launches += 1
        self._ops("sequential").coarse_correct(N, X_old, F_hat, G_cache, X_new, diff)

    def launch_count(self):
        return self.launches

    def set_profiling(self, on):
        pass

    def fine_stats(self):
        return dict(gemm_ms=0.0, gemm_flops=0.0, launches=0, other_ms=0.0)


class CpuBackend:
    name = "cpu-dryrun"
    dist_backend = "gloo"

    def __init__(self, local):
        self.device = torch.device("cpu")
        self.workload = None

    def init_dist(self, dist):
        dist.init_process_group("gloo")

    def sync(self):
        pass

    def event(self):
        return _Event()

    def make_context(self, P, systems, loads, J):
        import bench

        wl = bench.WORKLOADS[self.workload]
        return OracleContext(systems, loads, J, wl["T"], wl["N"], wl["alpha"])

    def clocks(self):
        return _NoClock()

    def flush_buffer(self):
        return torch.empty(8, dtype=torch.float64)

    def fp64_peak(self):
        return None
