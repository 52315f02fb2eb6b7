#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 Insum executor.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfgX] [--impl b200|reference]

Prints ONE JSON line (rank 0). A "step" is one pass of the hot path over one
batch of synthetic input: one indirect-Einsum evaluation (the evaluator
kernel) over operands already packed and resident in HBM. Workloads are the
BASELINE.json configs (see WORKLOADS); the default is configs[1], the
BlockGroupCOO SpMM on tcgen05 (falls back to configs[0] only if asked).

Timing: W untimed warm-up steps, then exactly K steps bracketed by a
barrier + cuda.synchronize on both sides; each step is bracketed by CUDA
events on the launching stream, with an L2 flush (256 MiB memset) between
steps outside the events; ms_per_step = mean; multi-GPU = max over ranks.
`e2e` re-times the same step through the public API with pinned host
buffers: H2D of the step's inputs + evaluation + D2H of the result.
`cpu_baseline` times the reference's own CPU path (oracle/_ref, the
unmodified reference compiled in place) on a bounded row slab of the same
matrix on this host.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "cfg2"
# L2 -> SM read bandwidth measured on this pool's B200s (tools/l2_rate.cu:
# 16-byte gathers of an L2-resident buffer, all SMs; profiles/l2_rate_r2.json)
L2_PEAK_GBPS = 21300.0
L2_PEAK_SOURCE = "measured tools/l2_rate.cu (profiles/l2_rate_r2.json)"


# --------------------------------------------------------------- helpers
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class Clocks:
    """Clock / throttle-reason sampler running DURING the timed region
    (B200_PROFILING.md clocks line). The kernels here run for tens of µs, so
    `nvidia-smi -lms 100` (one sample per 100 ms, ~200 ms start-up) sees none
    of them; this polls NVML (the library nvidia-smi reads) from a thread as
    fast as it answers, from start() to stop(). Falls back to nvidia-smi when
    pynvml is absent."""

    def __init__(self, torch_device):
        import threading
        self.samples = []  # (sm_mhz, reasons mask)
        self.max_mhz = None
        self.h = None
        self.nv = None
        self.p = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            try:
                import torch
                pr = torch.cuda.get_device_properties(torch_device)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(int(torch_device.index or 0))
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def _poll(self):
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(mhz), int(mask)))
            except Exception:
                return
            time.sleep(0.0005)

    def start(self):
        import threading
        if self.nv is not None:
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
        else:
            try:
                self.p = subprocess.Popen(
                    ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.p = None
        return self

    def stop(self):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)
        elif self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            for line in out.strip().splitlines():
                f = [x.strip() for x in line.split(",")]
                try:
                    self.samples.append((float(f[0]), int(f[2], 16)))
                    self.max_mhz = float(f[1])
                except (ValueError, IndexError):
                    continue
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"],
                    "samples_under_load": 0}
        sm, reasons = [], set()
        for mhz, mask in self.samples:
            if mask & 0x1:  # idle sample: not under load
                continue
            sm.append(mhz)
            for bit, name in REASONS.items():
                if mask & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples_under_load": len(sm),
                "samples": len(self.samples),
                "sampler": "nvml-thread" if self.nv is not None else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------- workloads
def time_builder(torch, fn, reps=10):
    """Wall time of a format-builder call (its plan phase syncs the host for
    the output sizes, so CUDA events would miss nothing but the host part):
    one warm call, then `reps` synchronised calls. Returns (result, ms) with
    ms = {"best": min, "median": median} over the reps."""
    out = fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return out, {"best": min(ts), "median": statistics.median(ts)}


class GroupCooWorkload:
    """configs[0] / configs[2]: unstructured GroupCOO SpMM, fp32 (K3)."""
    expr = "C[AM[p],n] = AV[p,q] * B[AK[p,q],n]"
    kernel = "spmm_groupcoo_kernel"

    def __init__(self, name, M, K, density, N, seed=1):
        self.name, self.M, self.K, self.density, self.N, self.seed = name, M, K, density, N, seed

    def config(self):
        return {"workload": self.name,
                "desc": f"GroupCOO SpMM fp32 {self.M}x{self.K} density {self.density} x N={self.N}",
                "expr": self.expr, "M": self.M, "K": self.K, "density": self.density,
                "N": self.N, "seed": self.seed}

    def setup(self, torch, P, S, dev, seed):
        rng = S.Rng(seed)
        # materialize order (driver.cpp:169-186): dense B first, then sparse A
        B = S.synth_dense(rng, (self.K, self.N), S.REAL, torch.float32)
        A = S.synth_sparse_matrix(rng, self.M, self.K, self.density, S.REAL, torch.float32)
        self.B = B.to(dev)
        Ad = A.to(dev)
        del A
        # K1 dense -> GroupCOO builder (format: auto, tuner on device), timed warm
        fmt, build_ms = time_builder(torch, lambda: P.dense_to_groupcoo(Ad, g=0))
        self.fmt = fmt
        self.G, self.g = fmt.num_groups(), fmt.group_size
        self.nnz = int(fmt.mask.sum().item())
        self.rows_nz = int(torch.unique(fmt.AM).numel())
        slots = self.G * self.g
        # builder: dense read (compulsory once; the kernels read it twice: count + pack)
        # + format written (AM, AK, AV, mask)
        self.builder = {"name": "K1 dense_to_groupcoo (+tuner)", "ms": build_ms["best"],
                        "ms_median": build_ms["median"],
                        "compulsory_bytes": self.M * self.K * 4 + self.G * 4 + slots * 9,
                        "passes_over_dense": 2}
        del Ad
        self.C = torch.empty((self.M, self.N), dtype=torch.float32, device=dev)
        self.flops = 2.0 * self.nnz * self.N
        # gather model (BASELINE §3): B row per stored nonzero + format
        # once + non-empty C rows once. It counts L2-served B rows as HBM bytes.
        self.alg_bytes = (self.nnz * self.N * 4 + slots * (4 + 4) + self.G * 4 +
                          self.rows_nz * self.N * 4)
        # compulsory DRAM: format once, B once, every C row written once (`=`)
        self.dram_bytes = self.G * 4 + slots * 8 + self.K * self.N * 4 + self.M * self.N * 4
        # L2 -> SM as the kernel moves it: one B row per slot (pads included) + format + C
        self.l2_bytes = self.G * 4 + slots * 8 + slots * self.N * 4 + self.M * self.N * 4
        self.tc_flops = None
        self.info = {"nnz": self.nnz, "G": self.G, "g": self.g, "nonempty_rows": self.rows_nz}
        # pinned host copies for e2e
        self.h_in = [fmt.AM.cpu().pin_memory(), fmt.AK.cpu().pin_memory(),
                     fmt.AV.cpu().pin_memory(), self.B.cpu().pin_memory()]
        self.h_out = torch.empty_like(self.C, device="cpu").pin_memory()
        self.d_in = [torch.empty_like(x, device=dev) for x in self.h_in]

    def step(self, P, stream=None):
        P.spmm_groupcoo(self.fmt.AM, self.fmt.AK, self.fmt.AV, self.B, self.C, accumulate=False,
                        flags=1 | 2)

    def e2e_step(self, P):
        # host buffers in, host C out: row-boundary chunks pipeline H2D / kernel / D2H
        AM, AK, AV, B = self.h_in
        P.spmm_groupcoo_host(AM, AK, AV, B, self.h_out, accumulate=False, nchunks=0)

    def e2e_bytes(self):
        return sum(x.numel() * x.element_size() for x in self.h_in), \
            self.h_out.numel() * self.h_out.element_size()

    def roofline_bound(self):
        return "hbm"

    # strong scaling through the native sharded C-ABI:
    # row-group shards of ONE replicated matrix, each rank writing its rows
    # of the full C, NCCL in-place broadcasts overlapping the next chunk
    def shard(self, torch, P, dev, rank, ws, comm=None, nchunks=4):
        from paper_2510_17505_b200 import distributed as D
        self.sh_plan = D.ShardPlan(self.fmt.AM, self.M, ws, rank, nchunks)
        self.sh_comm = comm
        self.C_full = torch.empty((self.M, self.N), dtype=torch.float32, device=dev)
        g0, _, r0, _ = self.sh_plan.chunk(rank, 0)
        _, g1, _, r1 = self.sh_plan.chunk(rank, nchunks - 1)
        return {"rows_owned": r1 - r0, "groups_owned": g1 - g0, "chunks": nchunks}

    def replicated(self):
        return [self.fmt.AM, self.fmt.AK, self.fmt.AV, self.B]

    def sharded_step(self, P, flags=0):
        from paper_2510_17505_b200 import distributed as D
        return D.spmm_groupcoo_sharded(self.sh_plan, self.fmt, self.B, self.C_full,
                                       self.sh_comm, flags=1 | 2 | flags)

    # reference CPU path on a bounded slab of the same matrix
    def cpu_sample(self, ref, budget_rows=None):
        # ~40M reference iteration points (G*g*N), ~1-2 s per reference run
        rows = budget_rows or int(4.0e7 / max(self.K * self.density * self.N, 1))
        rows = max(1, min(rows, self.M))
        rng = ref.Rng(self.seed)
        B = ref.synth_dense(rng, (self.K, self.N), 0)
        A = ref.synth_sparse_matrix(rng, rows, self.K, self.density, 0)  # first `rows` rows
        r, c, v = ref.dense_to_coo(A)
        import numpy as np
        g = ref.tune(np.bincount(r, minlength=rows))["chosen"]  # format: auto
        gc = ref.coo_to_groupcoo(rows, self.K, r, c, v, 0, g)
        t = {"AM": gc["AM"], "AK": gc["AK"], "AV": gc["AV"], "B": B}
        import numpy as np
        out = np.zeros((rows, self.N))
        return t, self.expr, "C", out, 2.0 * len(r) * self.N, f"first {rows} of {self.M} rows (nnz {len(r)}), g={g}"


class BlockGroupCooWorkload:
    """configs[1]: structured BlockGroupCOO SpMM, bf16 in / fp32 accumulate (K4, tcgen05)."""
    expr = "C[AM[p],bm,n] = AV[p,q,bm,bk] * B[AK[p,q],bk,n]"
    kernel = "bgcoo_tc_kernel"

    def __init__(self, name, M, K, b, bdens, N, seed=1):
        self.name, self.M, self.K, self.b, self.bdens, self.N, self.seed = \
            name, M, K, b, bdens, N, seed

    def config(self):
        return {"workload": self.name,
                "desc": f"BlockGroupCOO SpMM bf16 {self.M}x{self.K}, {self.b}x{self.b} blocks, "
                        f"{100 * (1 - self.bdens):.0f}% block sparsity x N={self.N}",
                "expr": self.expr, "M": self.M, "K": self.K, "block": self.b,
                "block_density": self.bdens, "N": self.N, "seed": self.seed}

    def setup(self, torch, P, S, dev, seed):
        rng = S.Rng(seed)
        b = self.b
        B = S.synth_dense(rng, (self.K // b, b, self.N), S.REAL, torch.bfloat16)
        A = S.synth_block_sparse_matrix(rng, self.M, self.K, b, b, self.bdens, S.REAL,
                                        torch.bfloat16)
        self.B = B.to(dev)
        Ad = A.to(dev)
        del A
        # K2 dense -> BlockGroupCOO builder (g by the tuner on block occupancy), timed warm
        fmt, build_ms = time_builder(torch, lambda: P.dense_to_blockgroupcoo(Ad, b, b, 0))
        del Ad
        self.fmt = fmt
        self.G, self.g = fmt.num_groups(), fmt.group_size
        self.nblk = fmt.num_blocks
        self.rows_nz = int(torch.unique(fmt.AM).numel())
        self.C = torch.empty((self.M // b, b, self.N), dtype=torch.float32, device=dev)
        self.flops = 2.0 * self.nblk * b * b * self.N
        slots = self.G * self.g
        # compulsory bytes: format once, dense operand once, C written once
        self.alg_bytes = (slots * b * b * 2 + slots * 4 + self.G * 4 + self.K * self.N * 2 +
                          self.rows_nz * b * self.N * 4)
        self.dram_bytes = slots * b * b * 2 + slots * 4 + self.G * 4 + self.K * self.N * 2 + \
            self.M * self.N * 4
        self.gather_bytes = slots * b * self.N * 2
        # L2 -> SM as the kernel moves it: a 16-row B tile per slot and n tile
        # (512 wide when N % 512 == 0), AV block + AK per slot and n tile, AM, C once
        ntile = self.N // 512 if self.N % 512 == 0 else max(self.N // 256, 1)
        self.l2_bytes = self.gather_bytes + slots * (b * b * 2 + 4) * ntile + self.G * 4 + \
            self.M * self.N * 4
        self.tc_flops = 2.0 * self.nblk * b * b * self.N
        # builder: dense read once + present blocks re-read + format written
        self.builder = {"name": "K2 dense_to_blockgroupcoo (+tuner)", "ms": build_ms["best"],
                        "ms_median": build_ms["median"],
                        "compulsory_bytes": self.M * self.K * 2 + self.nblk * b * b * 2 +
                        slots * (b * b * 2 + 4 + 1) + self.G * 4, "passes_over_dense": 1}
        self.mma_count = slots * (self.N // 128)  # one M=128 (n) x N=16 (bm) UMMA per slot per n tile
        self.info = {"blocks": self.nblk, "G": self.G, "g": self.g,
                     "nonempty_block_rows": self.rows_nz,
                     "gathered_B_tile_bytes": self.gather_bytes}
        self.h_in = [fmt.AM.cpu().pin_memory(), fmt.AK.cpu().pin_memory(),
                     fmt.AV.cpu().pin_memory(), self.B.cpu().pin_memory()]
        self.h_out = torch.empty_like(self.C, device="cpu").pin_memory()
        self.d_in = [torch.empty_like(x, device=dev) for x in self.h_in]

    def step(self, P, stream=None):
        P.spmm_blockgroupcoo(self.fmt.AM, self.fmt.AK, self.fmt.AV, self.B, self.C,
                             accumulate=False, flags=1 | 2)

    def e2e_step(self, P):
        # host buffers in, host C out: row-boundary chunks pipeline H2D / kernel / D2H
        AM, AK, AV, B = self.h_in
        P.spmm_blockgroupcoo_host(AM, AK, AV, B, self.h_out, accumulate=False, nchunks=0)

    def e2e_bytes(self):
        return sum(x.numel() * x.element_size() for x in self.h_in), \
            self.h_out.numel() * self.h_out.element_size()

    def roofline_bound(self):
        return "tensor"

    def shard(self, torch, P, dev, rank, ws, comm=None, nchunks=4):
        from paper_2510_17505_b200 import distributed as D
        self.sh_plan = D.ShardPlan(self.fmt.AM, self.M // self.b, ws, rank, nchunks)
        self.sh_comm = comm
        self.C_full = torch.empty_like(self.C)
        g0, _, r0, _ = self.sh_plan.chunk(rank, 0)
        _, g1, _, r1 = self.sh_plan.chunk(rank, nchunks - 1)
        return {"block_rows_owned": r1 - r0, "groups_owned": g1 - g0, "chunks": nchunks}

    def replicated(self):
        return [self.fmt.AM, self.fmt.AK, self.fmt.AV, self.B]

    def sharded_step(self, P, flags=0):
        from paper_2510_17505_b200 import distributed as D
        return D.spmm_blockgroupcoo_sharded(self.sh_plan, self.fmt, self.B, self.C_full,
                                            self.sh_comm, flags=1 | 2 | flags)

    def cpu_sample(self, ref, budget_rows=None):
        import numpy as np
        b = self.b
        brows = budget_rows or 8  # 1.6 % of the block rows: ~1 s per step on 8 host threads
        rng = ref.Rng(self.seed)
        B = ref.synth_dense(rng, (self.K // b, b, self.N), 0)
        A = ref.synth_block_sparse_matrix(rng, brows * b, self.K, b, b, self.bdens, 0)
        occ = (np.abs(A).reshape(brows, b, self.K // b, b).sum(axis=(1, 3)) > 0).sum(axis=1)
        g = ref.tune(occ)["chosen"]
        bg = ref.dense_to_blockgroupcoo(A, b, b, g, 0)
        nblk = int(bg["mask"].sum())
        t = {"AM": bg["AM"], "AK": bg["AK"], "AV": bg["AV"], "B": B}
        out = np.zeros((brows, b, self.N))
        return t, self.expr, "C", out, 2.0 * nblk * b * b * self.N, \
            f"first {brows} of {self.M // b} block rows ({nblk} blocks), g={g}"


class TensorProductWorkload:
    """configs[3]: e3nn-style CG tensor product, l_max 3, 64 channels, shared
    W[path,u,w] (K7, tcgen05). Metric: ms per call (lower is better)."""
    expr = "Z[b,CGI[p,q],w] = CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[CGL[p],u,w]"
    kernel = "tp_tc_kernel"
    metric = "TP ms/call"

    def __init__(self, name, batch, seed=1):
        self.name, self.batch, self.seed = name, batch, seed

    def config(self):
        return {"workload": self.name, "expr": self.expr,
                "desc": f"CG tensor product l_max=3 (23 paths, 353 real-basis CG nnz), 64 ch, "
                        f"batch {self.batch} edges, shared W, bf16 in / fp32 Z",
                "batch": self.batch, "seed": self.seed}

    def setup(self, torch, P, S, dev, seed):
        rng = S.Rng(seed)
        B = self.batch
        self.X = S.synth_dense(rng, (B, 16, 64), S.REAL, torch.bfloat16).to(dev)
        self.Y = S.synth_dense(rng, (B, 16), S.REAL, torch.bfloat16).to(dev)
        cg = S.cg_table(3)
        nl = cg["npaths"]
        self.W = S.synth_dense(rng, (nl, 64, 64), S.REAL, torch.bfloat16).to(dev)
        l = cg["l"].to(dev)
        g, _ = P.tune_group_size(l, nl)
        gt = P.group_coo_tensor([16, 16, 16, nl], [cg["i"].to(dev), cg["j"].to(dev),
                                                   cg["k"].to(dev), l], cg["v"].to(dev), 3, g)
        self.CGL, (self.CGI, self.CGJ, self.CGK), self.CGV = \
            gt.group_coord, gt.member_coords, gt.values
        import time as _t
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        # the CG table is validated and reshaped once (TpPlan), like ConvPlan for cfg5
        self.plan = P.TpPlan(self.CGL, self.CGI, self.CGJ, self.CGK, self.CGV, 16, 16, 16, nl)
        torch.cuda.synchronize()
        plan_ms = (_t.perf_counter() - t0) * 1e3
        self.Z = torch.empty((B, 16, 64), dtype=torch.float32, device=dev)
        self.flops = 2.0 * 99 * 64 * 64 * B  # factorised form (sum over paths of 2*l3+1 = 99)
        self.alg_bytes = B * (16 * 64 * 2 + 16 * 2 + 16 * 64 * 4) + nl * 64 * 64 * 2
        self.dram_bytes = self.alg_bytes
        # L2 -> SM: X/Y/Z once + W[l] (8 KB) per (pass, path) of the V-first schedule per
        # 64-edge tile (36 for the l_max = 3 table: 4 passes of 4 output rows)
        self.l2_bytes = self.alg_bytes + math.ceil(B / 64) * 36 * 64 * 64 * 2
        self.tc_flops = self.flops
        self.info = {"paths": nl, "cg_nnz": int(cg["v"].numel()), "G": gt.num_groups(), "g": g,
                     "plan_ms": plan_ms,
                     "formulation": "V-first: V[b,l,j,:] = X[b,j,:].W[l] on tcgen05 (99 (path, "
                                    "input component) products per edge, M=128 = 2 input rows x "
                                    "64 edges, A staged into TMEM by tcgen05.cp), Z = sum of "
                                    "(CG . Y) * V on CUDA cores in fp32"}
        self.h_in = [self.X.cpu().pin_memory(), self.Y.cpu().pin_memory()]
        self.h_out = torch.empty_like(self.Z, device="cpu").pin_memory()
        self.d_in = [torch.empty_like(x, device=dev) for x in self.h_in]

    def step(self, P, stream=None):
        self.plan.run(self.X, self.Y, self.W, self.Z, accumulate=False)

    def e2e_step(self, P):
        # host X/Y in, host Z out: edge chunks pipeline H2D / kernel / D2H
        self.plan.run_host(self.h_in[0], self.h_in[1], self.W, self.h_out, accumulate=False,
                           nchunks=8)

    def e2e_bytes(self):
        return sum(x.numel() * x.element_size() for x in self.h_in), \
            self.h_out.numel() * self.h_out.element_size()

    def roofline_bound(self):
        return "hbm"

    def units_total(self):
        return self.batch

    def shard(self, torch, P, dev, rank, ws, comm=None, nchunks=1):
        # edges are independent: each rank evaluates its edge block into its
        # own Z rows; Z stays sharded (no collective)
        from paper_2510_17505_b200 import distributed as D
        self.sh = D.edge_blocks(self.batch, ws)[rank]
        s = self.sh
        self.sh_X, self.sh_Y = self.X[s.r0:s.r1], self.Y[s.r0:s.r1]
        self.sh_Z = torch.empty((s.r1 - s.r0, 16, 64), dtype=torch.float32, device=dev)
        return {"edges_owned": s.r1 - s.r0, "collective": "none (Z stays sharded)"}

    def sharded_step(self, P, flags=0):
        if self.sh.r1 > self.sh.r0 and not flags & 16:
            self.plan.run(self.sh_X, self.sh_Y, self.W, self.sh_Z, accumulate=False)
        return self.sh_Z

    def cpu_sample(self, ref, budget_rows=None):
        import numpy as np
        from paper_2510_17505_b200 import synth as S
        cg = S.cg_table(3)
        nl = cg["npaths"]
        coords = np.stack([cg[k].numpy().astype(np.int64) for k in ("i", "j", "k", "l")])
        gt = ref.group_coo_tensor([16, 16, 16, nl], coords, cg["v"].double().numpy(), 3, 4)
        bs = budget_rows or 6
        rng = ref.Rng(self.seed)
        t = {"CGL": gt["group_coord"], "CGI": gt["member_coords"][0],
             "CGJ": gt["member_coords"][1], "CGK": gt["member_coords"][2], "CGV": gt["values"],
             "X": ref.synth_dense(rng, (bs, 16, 64), 0), "Y": ref.synth_dense(rng, (bs, 16), 0),
             "W": ref.synth_dense(rng, (nl, 64, 64), 0)}
        out = np.zeros((bs, 16, 64))
        return t, self.expr, "Z", out, bs, (f"{bs} of {self.batch} edges (same CG/W shapes, "
                                            f"own seed), extrapolated linearly to the batch")


class SparseConvWorkload:
    """configs[4]: submanifold 3x3x3 sparse conv, 1M voxels (sphere shells),
    C_in = C_out = 64, bf16 in / fp32 out (K5 kernel map + K6 on tcgen05).
    Metric: ms per call; the (output, offset) index of the map is built once
    (ConvPlan) outside the timed call and reported as plan_ms."""
    expr = "Out[MAPX[p,q],m] = MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]"
    kernel = "conv_tc_kernel"
    metric = "sparse-conv ms/call"

    def __init__(self, name, voxels, seed=1):
        self.name, self.voxels, self.seed = name, voxels, seed

    def config(self):
        return {"workload": self.name, "expr": self.expr,
                "desc": f"submanifold sparse conv 3x3x3, {self.voxels} voxels (sphere shells), "
                        f"C_in=C_out=64, bf16 in / fp32 out", "voxels": self.voxels,
                "seed": self.seed}

    def setup(self, torch, P, S, dev, seed):
        import time as _t
        coords = S.synth_voxel_shells(self.voxels).to(dev)
        n = coords.shape[0]
        def build():
            mo, mi, mz = P.kernel_map(coords)
            g, _ = P.tune_group_size(mz, 27)
            ones = torch.ones(mo.numel(), dtype=torch.float32, device=dev)
            return mo, mi, mz, g, P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g,
                                                     canonical=True)
        # K5 kernel map + tuner + group_coo_tensor, timed warm
        (mo, mi, mz, g, gt), build_ms = time_builder(torch, build)
        self.map, self.g = (mo, mi, mz), g
        self.MAPZ, (self.MAPX, self.MAPY), self.MAPV = gt.group_coord, gt.member_coords, gt.values
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        self.plan = P.ConvPlan(self.MAPZ, self.MAPX, self.MAPY, self.MAPV, n, 27, n)
        torch.cuda.synchronize()
        plan_ms = (_t.perf_counter() - t0) * 1e3
        rng = S.Rng(seed)
        self.In = S.synth_dense(rng, (n, 64), S.REAL, torch.bfloat16).to(dev)
        self.Wt = S.synth_dense(rng, (27, 64, 64), S.REAL, torch.bfloat16).to(dev)
        self.Out = torch.empty((n, 64), dtype=torch.float32, device=dev)
        pairs = mo.numel()
        self.pairs_total = pairs
        self.flops = 2.0 * pairs * 64 * 64
        G = gt.num_groups()
        # gather model: In row gathered + Out row updated per pair, map once
        self.alg_bytes = pairs * 64 * (2 + 4) + G * g * (4 + 2 * 4) + G * 4
        # compulsory DRAM: In once, Out once, the plan's input-row table Y[n, 28] int32
        self.dram_bytes = n * 64 * 2 + n * 64 * 4 + n * 28 * 4
        # L2 -> SM: an In row (128 B) per map pair, Weight[z] (8 KB) per used
        # (128-row tile, offset), the Y table, Out once
        tile_off = int(torch.unique((mo // 128).long() * 27 + mz.long()).numel())
        self.l2_bytes = pairs * 128 + tile_off * 64 * 64 * 2 + n * 28 * 4 + n * 64 * 4
        self.tc_flops = self.flops
        self.builder = {"name": "K5 kernel_map + tuner + group_coo_tensor", "ms": build_ms["best"],
                        "ms_median": build_ms["median"],
                        # coords read + hash table (2 x 8 B per slot) + pairs written (3 x 4 B)
                        # + grouped map written (MAPZ, MAPX, MAPY, MAPV)
                        "compulsory_bytes": n * 12 + 2 * n * 8 + pairs * 12 + G * 4 +
                        G * g * 12, "passes_over_dense": None}
        self.info = {"voxels": n, "pairs": pairs, "kappa": pairs / n, "G": G, "g": g,
                     "kernel_map_and_group_ms": build_ms["best"], "plan_ms": plan_ms}
        self.h_in = [self.In.cpu().pin_memory()]
        self.h_out = torch.empty_like(self.Out, device="cpu").pin_memory()
        self.d_in = [torch.empty_like(self.In)]

    def step(self, P, stream=None):
        self.plan.run(self.In, self.Wt, self.Out, accumulate=False)

    def e2e_step(self, P):
        # host In in, host Out out: output-tile chunks start as their input rows land
        self.plan.run_host(self.h_in[0], self.Wt, self.h_out, accumulate=False, nchunks=8)

    def e2e_bytes(self):
        return self.h_in[0].numel() * 2, self.h_out.numel() * 4

    def roofline_bound(self):
        return "hbm"

    def units_total(self):
        return getattr(self, "pairs_total", 9.12 * self.voxels)

    def shard(self, torch, P, dev, rank, ws, comm=None, nchunks=4):
        # point blocks: the map keeps only pairs whose output voxel is in the block
        import time as _t
        from paper_2510_17505_b200 import distributed as D
        n = self.In.shape[0]
        sh = D.point_blocks(n, ws)
        self.sh = sh[rank]
        self.sh_ws, self.sh_rank, self.sh_chunks, self.sh_comm = ws, rank, nchunks, comm
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        self.sh_plan = (D.conv_shard_plan(*self.map, n, self.sh, self.g)
                        if self.sh.r1 > self.sh.r0 else None)
        torch.cuda.synchronize()
        self.Out_full = torch.empty_like(self.Out)
        pairs = int(self.sh_plan.keep_map.mask.sum().item()) if self.sh_plan else 0
        return {"voxels_owned": self.sh.r1 - self.sh.r0, "pairs_owned": pairs,
                "chunks": nchunks, "shard_plan_ms": (_t.perf_counter() - t0) * 1e3}

    def replicated(self):
        return [self.In, self.Wt]

    def sharded_step(self, P, flags=0):
        from paper_2510_17505_b200 import distributed as D
        return D.conv_sharded(self.sh_plan, self.In, self.Wt, self.Out_full, self.sh_ws,
                              self.sh_rank, self.sh_chunks, self.sh_comm, flags=flags)

    def cpu_sample(self, ref, budget_rows=None):
        import numpy as np
        from oracle import ixo
        from paper_2510_17505_b200 import synth as S
        nv = budget_rows or 3000
        pts = S.synth_voxel_shells(nv).numpy()
        mo, mi, mz = ixo.kernel_map(pts)
        gt = ref.group_coo_tensor([nv, nv, 27], np.stack([mo, mi, mz]), np.ones(len(mo)), 2, 64)
        rng = ref.Rng(self.seed)
        t = {"MAPZ": gt["group_coord"], "MAPX": gt["member_coords"][0],
             "MAPY": gt["member_coords"][1], "MAPV": gt["values"],
             "In": ref.synth_dense(rng, (nv, 64), 0), "Weight": ref.synth_dense(rng, (27, 64, 64), 0)}
        out = np.zeros((nv, 64))
        return t, self.expr, "Out", out, len(mo), (
            f"first {nv} shell voxels ({len(mo)} map pairs), extrapolated linearly in pairs")


WORKLOADS = {
    "cfg1": lambda: GroupCooWorkload("cfg1", 4096, 4096, 0.01, 128),
    "cfg4": lambda: TensorProductWorkload("cfg4", 1_000_000),
    "cfg5": lambda: SparseConvWorkload("cfg5", 1_000_000),
    "cfg2": lambda: BlockGroupCooWorkload("cfg2", 8192, 8192, 16, 0.10, 512),
}
for _d in ("0.30", "0.20", "0.10", "0.05", "0.02"):
    WORKLOADS[f"cfg3_d{_d}"] = (lambda d: lambda: GroupCooWorkload(
        f"cfg3_d{d}", 16384, 16384, float(d), 256))(_d)

METRIC = "SpMM GFLOP/s (useful nnz)"


# ------------------------------------------------------------- arms
def cpu_reference_time(wl, steps=1, warmup=0, budget_rows=None):
    """Times the reference's CPU path (oracle/_ref) on a slab; returns dict."""
    from oracle import ref
    kind = "reference"
    if not ref.available():
        raise RuntimeError("oracle/_ref not built")
    t, expr, on, out, flops, sample = wl.cpu_sample(ref, budget_rows)
    cores = os.cpu_count() or 1
    # choose the faster reference path on this host: plan (1 core) vs the
    # threaded fused-lazy interpreter (kernel.cpp:1344-1411, all cores)
    modes = {}
    for mode, thr in (("plan", 1), ("fused-lazy", cores)):
        _, sc = ref.run(t, expr, on, out, mode, thr)
        modes[mode] = (sc["wall_ms"], thr)
    mode = min(modes, key=lambda m: modes[m][0])
    thr = modes[mode][1]
    for _ in range(warmup):
        ref.run(t, expr, on, out, mode, thr)
    times = []
    for _ in range(max(steps, 1)):
        _, sc = ref.run(t, expr, on, out, mode, thr)
        times.append(sc["wall_ms"])
    ms = statistics.mean(times)
    desc = (f"{sample}; reference execute_mode('{mode}', threads={thr}) "
            f"(plan {modes['plan'][0]:.1f} ms vs fused-lazy x{cores} "
            f"{modes['fused-lazy'][0]:.1f} ms)")
    if getattr(wl, "metric", METRIC) == METRIC:
        value, unit = flops / (ms * 1e-3) / 1e9, "GFLOP/s"
    else:  # time-like metric: the sample's time scaled to the whole call
        value, unit = ms * wl.units_total() / flops, "ms"
        desc += "; EXTRAPOLATED"
    return {"value": value, "unit": unit, "cores": thr, "kind": kind, "sample": desc,
            "ms_per_step": ms, "mode": mode}


def host_info():
    """CPU model and the reference build's compiler flags (BASELINE.md §5 asks
    for both next to every CPU number)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count(),
            "compiler": "g++ -std=c++20 -O2 (oracle/Makefile, unmodified reference sources)"}


def run_reference_arm(args, wl):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    r = cpu_reference_time(wl, steps=args.steps, warmup=args.warmup)
    metric = getattr(wl, "metric", METRIC)
    line = {"metric": metric, "value": r["value"], "unit": r["unit"], "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": metric == METRIC,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference synth, seed 1)", "config": wl.config(),
            "cpu_baseline": {"value": r["value"], "unit": r["unit"], "cores": r["cores"],
                             "kind": r["kind"], "sample": r["sample"], **host_info()},
            "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_ncu_traffic(name):
    path = os.path.join(ROOT, "profiles", f"ncu_{name}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def roofline(wl, kern_s, torch, dev):
    """Three fractions of the step's dominant kernel:
    compulsory DRAM bytes vs measured HBM, the kernel's L2->SM bytes vs the
    measured L2 read bandwidth, and tensor-core flops vs measured bf16 peak
    (tensor-core kernels only). `bound` is the binding level: the one whose
    floor (bytes or flops / peak) is longest, i.e. the largest fraction."""
    hbm, tc, _, peak_src = load_peaks()
    fr = {"hbm": wl.dram_bytes / kern_s / 1e9 / hbm,
          "l2": wl.l2_bytes / kern_s / 1e9 / L2_PEAK_GBPS}
    if wl.tc_flops:
        fr["tensor"] = wl.tc_flops / kern_s / 1e12 / tc
    bound = max(fr, key=fr.get)
    if bound == "tensor":
        achieved, peak, unit = wl.tc_flops / kern_s / 1e12, tc, "TFLOP/s"
        src = f"{peak_src} MEASURED_PEAKS.json bf16_tflops (burst)"
    elif bound == "hbm":
        achieved, peak, unit = wl.dram_bytes / kern_s / 1e9, hbm, "GB/s"
        src = f"{peak_src} MEASURED_PEAKS.json hbm_gbs"
    else:
        achieved, peak, unit = wl.l2_bytes / kern_s / 1e9, L2_PEAK_GBPS, "GB/s"
        src = L2_PEAK_SOURCE
    roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": load_ncu_traffic(wl.name),
            "traffic_source": f"profiles/ncu_{wl.name}.json (ncu --set full, dram__bytes "
                              "read+write per launch)",
            "fracs": fr, "peak_source": src,
            "bytes": {"dram_compulsory": wl.dram_bytes, "l2_to_sm": wl.l2_bytes},
            "tc_flops": wl.tc_flops,
            "peaks": {"hbm_GBps": hbm, "l2_GBps": L2_PEAK_GBPS, "bf16_TFLOPs": tc}}
    if hasattr(wl, "alg_bytes") and wl.roofline_bound() == "hbm":
        # BASELINE §3's gather model (B rows counted as if from HBM)
        roof["gather_model_frac"] = wl.alg_bytes / kern_s / 1e9 / hbm
    if hasattr(wl, "mma_count"):
        # measured tensor-pipe occupancy of an M=128,N=16,K=16 MMA with >= 2 issuing CTAs
        # per SM: 38.8 cycles (tools/umma_pair_rate.cu, profiles/k4_diag_r1.md §8 and
        # k4_diag_r2.md §1); the per-instruction floor, not flops, bounds 16-wide blocks
        floor_s = wl.mma_count * 38.8 / (torch.cuda.get_device_properties(dev).multi_processor_count
                                          * 1.965e9)
        roof["mma_issue_floor_us"] = floor_s * 1e6
        roof["frac_of_mma_issue_floor"] = floor_s / kern_s
    return roof


def measure(torch, P, step, e2e_step, steps, warmup, e2e_reps, flush, stream, graph=True,
            ws=1, dist=None):
    """W warm-up steps, then `steps` timed steps (CUDA-graph replay of one
    step unless graph=False), each bracketed by events on `stream` after an
    L2 flush outside the events; clocks sampled during the timed region;
    max over ranks. Then the e2e leg through the public API."""
    dev = flush.device
    for _ in range(warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    P.lib().ixb_check_errors(None)
    timed_step, timing, per_step = step, "eager launches", None
    if graph:
        try:
            c0 = P.lib().ixb_launch_count()
            g = torch.cuda.CUDAGraph()
            # thread_local: CUDA calls from other threads (NCCL's) during the
            # capture neither fail nor invalidate it
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                step()
            per_step = P.lib().ixb_launch_count() - c0
            g.replay()
            torch.cuda.synchronize()
            timed_step, timing = g.replay, "CUDA-graph replay of one step"
        except Exception as e:  # reported in config.timing, never fatal
            timing = f"eager launches (graph capture failed: {type(e).__name__})"
            torch.cuda.synchronize()
    clocks = Clocks(dev)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = P.lib().ixb_launch_count()
    evs = []
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        timed_step()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = P.lib().ixb_launch_count() - launches0
    if per_step is not None:
        launches = per_step * steps
    clk = clocks.stop()
    rc = P.lib().ixb_check_errors(None)
    if rc != 0:
        raise RuntimeError("index error during bench: " + P.lib().ixb_last_error().decode())
    total = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([total], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item() / steps
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e_evs = []
    for _ in range(e2e_reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        e_evs.append((a, b))
    torch.cuda.synchronize()
    # median over the reps (host-side hiccups in a rep of a sub-ms call
    # otherwise dominate a mean); the mean is reported beside it
    e_all = [a.elapsed_time(b) for a, b in e_evs]
    e_ms = statistics.median(e_all)
    e_mean = statistics.mean(e_all)
    et = torch.tensor([e_ms, e_mean], device=dev, dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    return {"ms": ms, "e2e_ms": et[0].item(), "e2e_mean_ms": et[1].item(),
            "launches": int(launches), "timing": timing, "clocks": clk}


def workload_record(wl, m, torch, dev, jobs=1, kern_scale=1.0):
    """The JSON fields of one workload measured by `measure`."""
    metric = getattr(wl, "metric", METRIC)
    timelike = metric != METRIC
    ms = m["ms"]
    value = wl.flops * jobs / (ms * 1e-3) / 1e9
    h2d, d2h = wl.e2e_bytes() if hasattr(wl, "e2e_bytes") else (None, None)
    rec = {"metric": metric, "value": ms if timelike else value,
           "unit": "ms" if timelike else "GFLOP/s", "ms_per_step": ms,
           "higher_is_better": not timelike,
           "dtype": "bf16" if wl.tc_flops or timelike else "f32",
           "config": dict(wl.config(), timing=m["timing"], **wl.info),
           "roofline": roofline(wl, ms * 1e-3 * kern_scale, torch, dev),
           "clocks": m["clocks"], "gpu_launches": m["launches"],
           "e2e": {"value": m["e2e_ms"] if timelike else wl.flops * jobs / (m["e2e_ms"] * 1e-3) / 1e9,
                   "unit": "ms" if timelike else "GFLOP/s", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": m["e2e_ms"],
                   "aggregate": "median of reps", "mean_ms": m["e2e_mean_ms"]}}
    if timelike:
        rec["config"]["useful_GFLOPs"] = value
    return rec


def builder_record(wl):
    """Format-builder timing recorded by the workload's setup (warm call)."""
    hbm, _, _, _ = load_peaks()
    b = dict(wl.builder)
    gbps = b["compulsory_bytes"] / (b["ms"] * 1e-3) / 1e9
    b.update({"workload": wl.name, "achieved_GBps": gbps, "hbm_frac": gbps / hbm,
              "timing": "wall time of the API call (warm, best of 10, median beside it; its plan "
                        "phase syncs the host for the output sizes)"})
    return b


def cpu_builder_baseline(name):
    """The reference's own builders on the same full-size input (cfg1: dense_to_coo +
    tune + coo_to_groupcoo; cfg2: dense_to_blockgroupcoo), oracle/_ref, one core."""
    import numpy as np
    from oracle import ref
    if not ref.available():
        return None
    if name == "cfg1":
        rng = ref.Rng(1)
        ref.synth_dense(rng, (4096, 128), 0)
        A = ref.synth_sparse_matrix(rng, 4096, 4096, 0.01, 0)
        t0 = time.perf_counter()
        r, c, v = ref.dense_to_coo(A)
        g = ref.tune(np.bincount(r, minlength=4096))["chosen"]
        ref.coo_to_groupcoo(4096, 4096, r, c, v, 0, g)
        ms = (time.perf_counter() - t0) * 1e3
        return {"ms": ms, "cores": 1, "kind": "reference",
                "sample": "full cfg1 matrix: dense_to_coo + tuner + coo_to_groupcoo"}
    if name == "cfg2":
        rng = ref.Rng(1)
        ref.synth_dense(rng, (512, 16, 512), 0)
        A = ref.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, 0)
        t0 = time.perf_counter()
        ref.dense_to_blockgroupcoo(A, 16, 16, 8, 0)
        ms = (time.perf_counter() - t0) * 1e3
        return {"ms": ms, "cores": 1, "kind": "reference",
                "sample": "full cfg2 matrix: dense_to_blockgroupcoo (g=8, the tuner's choice)"}
    return None


SECONDARY = ["cfg1", "cfg3_d0.30", "cfg3_d0.20", "cfg3_d0.10", "cfg3_d0.05", "cfg3_d0.02",
             "cfg4", "cfg5"]
# bounded reference samples for the secondary workloads (a few seconds each)
SECONDARY_BUDGET = {"cfg1": 1000, "cfg4": 2, "cfg5": 800}
for _d in (0.30, 0.20, 0.10, 0.05, 0.02):  # ~2e7 reference iteration points per run
    SECONDARY_BUDGET[f"cfg3_d{_d:.2f}"] = max(1, int(2.0e7 / (16384 * _d * 256)))


def run_b200(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2510_17505_b200 as P
    from paper_2510_17505_b200 import synth as S

    ws, rank, local = dist_env()
    # IXB_DIST_BACKEND=gloo lets several ranks share one GPU: a functional
    # check of the sharded path on a 1-GPU box, never a timing
    backend = os.environ.get("IXB_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    P.lib()
    if args.sharded:
        # strong scaling: every rank holds the SAME instance
        # and runs the native sharded C-ABI path (its rows of the full
        # output, NCCL in-place broadcasts overlapping the next chunk)
        from paper_2510_17505_b200 import distributed as D
        wl.setup(torch, P, S, dev, wl.seed)
        comm = D.Comm(ws, rank) if ws > 1 else None
        shard_info = wl.shard(torch, P, dev, rank, ws, comm)

        def step():
            wl.sharded_step(P)

        out_t = wl.sharded_step(P)
        h_out = torch.empty(out_t.shape, dtype=out_t.dtype).pin_memory()

        def e2e_step():
            # inputs are replicated once (outside the step); the result read back
            h_out.copy_(wl.sharded_step(P), non_blocking=True)

        def e2e_bytes():
            return 0, h_out.numel() * h_out.element_size()
        wl.e2e_bytes = e2e_bytes
    else:
        # weak scaling: every rank evaluates its own independent instance of the
        # per-GPU workload (seed + rank); no data-path collective.
        wl.setup(torch, P, S, dev, wl.seed + rank)
        shard_info = None

        def step():
            wl.step(P)

        def e2e_step():
            wl.e2e_step(P)
    jobs = 1 if args.sharded else ws  # instances processed per step, whole job
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    m = measure(torch, P, step, e2e_step, args.steps, args.warmup, max(3, min(args.steps, 20)),
                flush, stream, graph=not args.no_graph, ws=ws, dist=dist)
    rec = workload_record(wl, m, torch, dev, jobs=jobs,
                          kern_scale=ws if args.sharded else 1)
    line = {"metric": rec["metric"], "value": rec["value"], "unit": rec["unit"], "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
            "higher_is_better": rec["higher_is_better"],
            "scaling": "strong" if args.sharded else "weak", "vs_baseline": None,
            "dtype": rec["dtype"], "data": "synthetic (reference synth streams, seed 1 + rank)",
            "config": dict(rec["config"], l2="flushed between steps (256 MiB memset outside "
                                             "the timed events)",
                           parallelism=(f"sharded x{ws} + {'NCCL in-place broadcast' if ws > 1 else 'no'} "
                                        "all-gather of output rows"
                                        if args.sharded else f"weak x{ws} (independent replicas)")),
            "roofline": rec["roofline"], "clocks": rec["clocks"],
            "gpu_launches": rec["gpu_launches"], "e2e": rec["e2e"]}
    if shard_info is not None:
        line["config"]["shard_rank0"] = shard_info
    if ws > 1:
        line["config"]["dist_backend"] = backend
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_line(wl)
    builders = {}
    if getattr(wl, "builder", None) and not args.sharded:
        builders[wl.name] = builder_record(wl)
    if not args.sharded and not args.no_sharded_records:
        line["sharded"] = sharded_records(torch, P, S, dev, rank, ws, dist, flush, stream,
                                          args.sub_steps)
    if ws == 1 and not args.sharded and args.workloads != "none":
        # every other BASELINE config, measured the same way in this invocation
        names = SECONDARY if args.workloads == "all" else args.workloads.split(",")
        line["workloads"] = {}
        del wl
        for name in names:
            if name == args.workload:
                continue
            w2 = WORKLOADS[name]()
            try:
                w2.setup(torch, P, S, dev, w2.seed)
                m2 = measure(torch, P, lambda: w2.step(P), lambda: w2.e2e_step(P),
                             args.sub_steps, 3, 3, flush, stream, graph=not args.no_graph)
                r2 = workload_record(w2, m2, torch, dev)
                r2["steps"], r2["warmup"] = args.sub_steps, 3
                if not args.no_cpu_baseline:
                    r2["cpu_baseline"] = cpu_line(w2, SECONDARY_BUDGET.get(name), steps=1)
                if getattr(w2, "builder", None):
                    builders[name] = builder_record(w2)
                line["workloads"][name] = r2
            except Exception as e:  # reported per workload, never fatal to the headline
                line["workloads"][name] = {"error": f"{type(e).__name__}: {e}"}
            del w2
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    if builders:
        if not args.no_cpu_baseline:
            for name, b in builders.items():
                cb = cpu_builder_baseline(name)
                if cb:
                    b["cpu_baseline"] = cb
        line["builders"] = builders
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


SHARDED = ["cfg3_d0.30", "cfg5"]  # BASELINE configs[2] and [4]: "sharded 1/2/4/8 B200"


def time_graph(torch, step, steps, flush, stream, ws, dist):
    """Mean ms of `steps` CUDA-graph replays of `step` (L2 flushed outside the
    events, as in measure), max over ranks."""
    for _ in range(3):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        step()
    g.replay()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    evs = []
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / steps], dtype=torch.float64,
                     device=flush.device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def sharded_records(torch, P, S, dev, rank, ws, dist, flush, stream, steps, names=SHARDED):
    """Strong scaling of the BASELINE "sharded 1/2/4/8" configs through the
    native sharded C-ABI: every rank holds the same instance
    and evaluates its row-group / point-block shard in 4 chunks into its rows
    of the full output; chunk c's NCCL in-place broadcasts overlap chunk
    c+1's kernel. Reported per N: the whole step, the compute alone (no
    collective) and the all-gather alone, each max over ranks; at N = 1 also
    the unsharded evaluator for the sharding overhead."""
    from paper_2510_17505_b200 import distributed as D
    comm = D.Comm(ws, rank) if ws > 1 else None
    out = {}
    for name in names:
        wl = WORKLOADS[name]()
        try:
            wl.setup(torch, P, S, dev, wl.seed)  # same seed: one instance, replicated
            if comm is not None:  # rank 0's operands are the ones every rank uses
                comm.broadcast(*wl.replicated())
                torch.cuda.synchronize()
            # chunks only buy overlap with the all-gather: one chunk without it
            info = wl.shard(torch, P, dev, rank, ws, comm, nchunks=4 if ws > 1 else 1)
            total = time_graph(torch, lambda: wl.sharded_step(P), steps, flush, stream, ws, dist)
            compute = time_graph(torch, lambda: wl.sharded_step(P, D.SHARD_NO_COMM), steps,
                                 flush, stream, ws, dist)
            gather = (time_graph(torch, lambda: wl.sharded_step(P, D.SHARD_COMM_ONLY), steps,
                                 flush, stream, ws, dist) if comm is not None else 0.0)
            timelike = getattr(wl, "metric", METRIC) != METRIC
            rec = {"metric": getattr(wl, "metric", METRIC), "unit": "ms" if timelike else "GFLOP/s",
                   "value": total if timelike else wl.flops / (total * 1e-3) / 1e9,
                   "ms_per_step": total, "compute_ms": compute, "gather_ms": gather,
                   "overlap": (compute + gather - total) / gather if gather > 0 else None,
                   "n_gpus": ws, "scaling": "strong", "steps": steps,
                   "config": dict(wl.config(), **wl.info, shard_rank0=info if rank == 0 else None,
                                  parallelism=f"sharded x{ws}" + (
                                      " + NCCL in-place broadcast all-gather of output rows, "
                                      "overlapped by chunk" if ws > 1 else " (no collective)"),
                                  timing="CUDA-graph replay, max over ranks, L2 flushed")}
            rec["useful_GFLOPs"] = wl.flops / (total * 1e-3) / 1e9
            if ws == 1:
                rec["unsharded_ms"] = time_graph(torch, lambda: wl.step(P), steps, flush, stream,
                                                 ws, dist)
                rec["sharding_overhead"] = total / rec["unsharded_ms"] - 1.0
            out[name] = rec
        except Exception as e:  # reported per workload, never fatal to the headline
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        del wl
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    return out


def cpu_line(wl, budget=None, steps=1):
    try:
        r = cpu_reference_time(wl, steps=steps, budget_rows=budget)
        return dict({k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}, **host_info())
    except Exception as e:  # reported, never fatal
        return {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "reference",
                "sample": f"unavailable: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of a CUDA-graph replay of the step")
    ap.add_argument("--workloads", default="all",
                    help="other BASELINE configs timed in the same invocation (N=1 only): "
                         "'all', 'none' or a comma list")
    ap.add_argument("--sub-steps", type=int, default=10,
                    help="timed steps per secondary workload")
    ap.add_argument("--no-sharded-records", action="store_true",
                    help="skip the strong-scaling records of the sharded BASELINE configs")
    ap.add_argument("--sharded", action="store_true",
                    help="strong scaling: shard ONE instance across the ranks (row groups, "
                         "point blocks or edges) and all-gather the output inside the step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]()
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_b200(args, wl)


if __name__ == "__main__":
    main()
