#!/usr/bin/env python
"""Benchmark of the B200 QR-TEBD bond update (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config north] [--impl ours|reference]

Workload (default at N=1: the north-star configuration of BASELINE.json,
SURVEY.md §8(d) "North-star target"): global quench of the d=5 quantum clock
model, uniform MPS with unit cell L=2, chi=1024, QR truncation (chi_max = chi,
so eta = chi), complex128, Trotter order 2 (3 dependent two-site updates per
step), g=2, dt=0.05, explicit truncation error on (the quench default,
proj/include/qrtebd/gates.hpp:51).  Synthetic steady-state input at fixed
chi: random right isometries and a Gaussian bond matrix (the bench_cell
recipe, proj/src/run.cpp:345-381).  theta = 419 MB, far larger than L2.

A "step" is one tebd_step (proj/src/gates.cpp:513-540) with the state
resident in HBM (device-resident UniformMPS, one CUDA-graph replay per
step).  `value` = Trotter steps/s; `e2e` = the same metric with the state
copied host->device from pinned memory before and device->host after every
step; `roofline` = the whole step's algorithmic flops per
second against the FP64 DMMA peak measured in the run.

The uniform cell does not shard (3 strictly dependent updates, a single bond
is never split).  Under torchrun with N > 1 and no --config the default
workload is the C5 finite chain (BASELINE.json configs[4]: N=256 sites,
chi=512), sites sharded over the ranks with boundary exchange (strong
scaling); --config <uniform cell> with N > 1 runs N replicas.

--impl reference times the reference algorithm on the host CPU (the
NumPy/LAPACK oracle port, oracle/qrtebd_oracle.py) on the
same config, as a bounded sample of single bond updates.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# every complex product on the tensor pipe is 3M (Gauss): three real DMMAs per
# complex 8x8x4 step (csrc/zgemm.cu), so algorithmic flops (8 per complex
# MAC) can run above the 4-product DMMA peak; the method's own
# ceiling is 4/3 of it (peak_3m)
COMPLEX_3M_NOTE = ("3M complex products (three real DMMA per complex MAC): algorithmic flops / DMMA peak may exceed 1; "
                   "frac_of_3m_peak is against 4/3 x the DMMA peak, the method's tensor-pipe ceiling")
METRIC = "Trotter steps/sec (2-site QR updates/sec) vs chi,d; FP64 tensor-pipe % of peak"

CONFIGS = {
    # name: (description, d, chi, scheme, explicit error, (delta_chi_abs, delta_chi_rel))
    "c1": ("C1 iTEBD transverse-field Ising (clock d=2), L=2, chi=64, qr", 2, 64, "qr", True, (0, 0.0)),
    "c2": ("C2 clock-model quench d=5, chi=256, uniform L=2, qr (eta=chi), explicit error on", 5, 256, "qr", True,
           (0, 0.0)),
    "c2cbe": ("C2 clock-model quench d=5, chi=256, uniform L=2, qr_cbe (eta=356 -> 256), explicit error on", 5, 256,
              "qr_cbe", True, (100, 0.1)),
    "north": ("north-star clock quench d=5, chi=1024, uniform L=2, qr (eta=chi), explicit error on", 5, 1024, "qr",
              True, (0, 0.0)),
    "northcbe": ("north-star clock quench d=5, chi=1024, uniform L=2, qr_cbe (eta=1127 -> 1024), explicit on", 5,
                 1024, "qr_cbe", True, (100, 0.1)),
    "c3": ("C3 clock d=10, chi=1024, uniform L=2, qr_cbe (eta=1127 -> 1024), explicit error on", 10, 1024, "qr_cbe",
           True, (100, 0.1)),
    "c4": ("C4 single-bond stress d=5, chi=4096, qr bench cell (eta=chi, explicit off), 3 updates per step", 5, 4096,
           "qr", False, (0, 0.0)),
}


CHAIN_CONFIGS = {
    # finite open chain, Hastings form, sites sharded over the ranks
    "c5": dict(desc="C5 finite clock chain N=256, d=5, chi=512, qr, even/odd bonds sharded over ranks "
                    "(NCCL send/recv of boundary tensors), explicit error on",
               n=256, d=5, chi=512, scheme="qr", explicit=True),
    "c5small": dict(desc="finite clock chain N=32, d=3, chi=64, qr (smoke-size C5)", n=32, d=3, chi=64, scheme="qr",
                    explicit=True),
}


def policy_kw(cfg):
    _, d, chi, scheme, explicit, (dabs, drel) = cfg
    return dict(chi_max=chi, delta_chi_abs=dabs, delta_chi_rel=drel, compute_explicit_error=explicit)


def widths(cfg):
    """(eta, kk) of the steady-state update (gates.cpp:94-101, :354-355, :398-419)."""
    _, d, chi, scheme, _, (dabs, drel) = cfg
    eta = min(d * chi, chi + max(dabs, math.ceil(drel * chi)))
    if scheme == "qr":
        eta = min(eta, chi)
    return eta, chi


def flops_per_update(d, chi, eta, kk, explicit, cbe=False):
    """8 flops per complex MAC; eigh excluded for CBE."""
    f = 8.0 * (2 * d * d * chi ** 3 + d ** 4 * chi ** 2 + 2 * d * d * chi * chi * eta + d * d * chi * chi * kk)
    f += 2.0 * (16.0 * (d * chi) * eta * eta - 16.0 / 3.0 * eta ** 3)
    if explicit:
        f += 8.0 * (eta * eta * d * chi + d * d * chi * chi * eta)
    if cbe:
        f += 8.0 * (eta ** 3 + kk * eta * d * chi)
        if explicit:
            f += 8.0 * (eta * eta * kk + eta ** 3)
    return f


def synthetic_state(d, chi, seed=0x51AB):
    """Random right-canonical L=2 state at fixed chi (bench_cell recipe)."""
    rng = np.random.default_rng([seed, d, chi])

    def right_iso():
        g = rng.standard_normal((d * chi, chi)) + 1j * rng.standard_normal((d * chi, chi))
        q, r = np.linalg.qr(g)  # columns orthonormal -> rows of q^H orthonormal
        q = q * (np.diag(r) / np.abs(np.diag(r)))
        qh = q.conj().T  # (chi, d*chi) with orthonormal rows
        return np.ascontiguousarray(qh.reshape(chi, d, chi).transpose(1, 0, 2))

    def bond():
        x = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
        return x / np.linalg.norm(x)

    return [right_iso(), right_iso()], [bond(), bond()]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        # in-process NVML (the same counters nvidia-smi reads): spawning
        # nvidia-smi every 200 ms held driver locks long enough to stall the
        # launching thread and showed up as idle time inside the event pairs
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            pynvml = None
        while not self._stop.is_set():
            try:
                if pynvml is not None:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                             pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
                    self.samples.append([str(sm), str(mx)] + ["Active" if rs & f else "Not Active" for f in flags])
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.02)  # ~50 samples/s: several inside even a short timed region

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 2 + k and s[2 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def host_info():
    """CPU model, sockets, cores and NUMA nodes of the host the CPU baseline ran on."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        model, phys = None, set()
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("physical id"):
                    phys.add(ln.split(":", 1)[1].strip())
        info["model"] = model
        info["sockets"] = len(phys) or None
        info["numa_nodes"] = len([x for x in os.listdir("/sys/devices/system/node") if x.startswith("node")])
    except OSError:
        pass
    return info


def cpu_reference_rate(cfg, budget_s, min_updates=1, warmup_updates=0, seed=0x51AB, scheme=None):
    """Reference algorithm on the host cores (the oracle port: test infra,
    never the measured product).  Times single bond updates in Trotter order
    on the evolving L=2 state (even dt/2, odd dt, even dt/2, ...); a Trotter
    step is exactly 3 updates and nothing else (proj/src/gates.cpp:513-540),
    so steps/s = (updates / 3) / elapsed.  Bounded sample: stops after
    `min_updates` once `budget_s` has elapsed (at least one update).
    Returns (steps/s, updates timed, seconds)."""
    from oracle import qrtebd_oracle as ref
    from paper_2212_09782_b200 import model
    _, d, chi, cfg_scheme, _, _ = cfg
    scheme = scheme or cfg_scheme
    sites, bonds = synthetic_state(d, chi, seed)
    sites, bonds = [x.copy() for x in sites], [x.copy() for x in bonds]
    gates = [model.make_gate(model.bond_hamiltonian(d, 2.0), dte) for _, dte in model.layer_structure(0.05, 2)]
    pol = ref.TruncationPolicy(**policy_kw(cfg))
    k = 0

    def one_update():
        nonlocal k
        layer = k % 3
        m = 0 if layer != 1 else 1  # L = 2: even bond (0,1), odd bond (1,0)
        n = 1 - m
        upd = ref.apply_gate(scheme, bonds[m], sites[m], sites[n], gates[layer], pol)
        sites[m], bonds[n], sites[n] = upd.b_m, upd.xi_n, upd.b_n
        k += 1

    for _ in range(warmup_updates):
        one_update()
    n, t0 = 0, time.perf_counter()
    while True:
        one_update()
        n += 1
        if n >= min_updates and time.perf_counter() - t0 >= budget_s:
            break
        if budget_s > 0 and time.perf_counter() - t0 >= 4 * budget_s:
            break
    dt = time.perf_counter() - t0
    return (n / 3.0) / dt, n, dt


REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


def reference_binary_rate(cfg, budget_s, min_updates=1, scheme=None):
    """The reference ITSELF on the host cores: oracle/_ref/ref_bench is
    /root/reference/proj/src compiled in place on the Eigen-3.4-subset shim
    over OpenBLAS (oracle/Makefile; test infrastructure, never the product).
    It runs the reference's own apply_gate in tebd_step order on the same
    synthetic state, with the reference's own gate construction, all host
    threads.  Returns (steps/s, updates, seconds, threads) or None when the
    binary is absent."""
    import tempfile
    if not os.access(REF_BENCH, os.X_OK):
        return None
    _, d, chi, cfg_scheme, explicit, (dabs, drel) = cfg
    sites, bonds = synthetic_state(d, chi)
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "state.bin")
        with open(path, "wb") as f:
            for a in sites + bonds:
                f.write(np.ascontiguousarray(a, dtype=np.complex128).tobytes())
        # the reference is built without OpenMP (oracle/Makefile): its products
        # run on the OpenBLAS pool, all host cores
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(cores))
        out = subprocess.run([REF_BENCH, path, str(d), str(chi), scheme or cfg_scheme, "1" if explicit else "0",
                              str(dabs), str(drel), str(budget_s), str(min_updates)], capture_output=True, text=True,
                             env=env)
    if out.returncode != 0:
        raise RuntimeError(f"ref_bench failed: {out.stderr[-500:]}")
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return (r["updates"] / 3.0) / r["seconds"], r["updates"], r["seconds"], r["threads"]


def config_dict(cfg, ws):
    """The `config` object both arms print (identical keys and values)."""
    desc, d, chi, scheme, explicit, _ = cfg
    eta, _ = widths(cfg)
    return {"workload": desc, "d": d, "chi": chi, "eta": eta, "scheme": scheme, "cell_length": 2,
            "explicit_error": explicit, "trotter_order": 2, "updates_per_step": 3,
            "parallelism": f"replicas x{ws}" if ws > 1 else "single",
            "l2": "flushed (256 MB write) between timed steps, outside the per-step event pair"}


def run_reference(args, cfg):
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    desc, d, chi, scheme, explicit, _ = cfg
    cores = os.cpu_count()
    # bounded sample: K steps' worth of updates on small cells; on large cells
    # (north star: ~10 s per update on 16 cores) as many updates as fit in
    # the budget, at least one -- the whole run stays within a few minutes
    budget = float(os.environ.get("QT_REF_BUDGET_S", "60"))
    kind = os.environ.get("QT_REF_IMPL", "reference")
    refbin = reference_binary_rate(cfg, budget_s=budget if chi > 256 else 0.0,
                                   min_updates=3 * max(1, args.steps) if chi <= 256 else 1) \
        if kind == "reference" else None
    if refbin is not None:
        rate, n, dt, cores = refbin
        sample = (f"{n} bond updates ({n / 3:.2f} Trotter steps, {dt:.1f} s) of the reference itself "
                  f"(proj/src compiled in place on the Eigen-3.4-subset shim over OpenBLAS LAPACK, "
                  f"oracle/_ref/ref_bench) in tebd_step order on the same synthetic state, {cores} threads; "
                  "steps/s = updates/3 / time")
        kind = "reference"
    else:
        warm = 1 if (args.warmup > 0 and chi <= 256) else 0
        rate, n, dt = cpu_reference_rate(cfg, budget_s=budget if chi > 256 else 0.0,
                                         min_updates=3 * max(1, args.steps) if chi <= 256 else 1, warmup_updates=warm)
        sample = (f"{n} bond updates ({n / 3:.2f} Trotter steps, {dt:.1f} s) of the NumPy/LAPACK oracle port in "
                  f"Trotter order on the same synthetic state and gates (OpenBLAS, {cores} threads); steps/s = "
                  "updates/3 / time")
        kind = "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / rate, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
        "config": config_dict(cfg, 1),
        "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": cores, "kind": kind, "sample": sample,
                         "host": host_info()},
        "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def chain_config_dict(cc, ws):
    """The `config` object both arms print for a finite chain."""
    n = cc["n"]
    upd = 2 * len(range(0, n - 1, 2)) + len(range(1, n - 1, 2))
    return {"workload": cc["desc"], "n_sites": n, "d": cc["d"], "chi": cc["chi"], "scheme": cc["scheme"],
            "explicit_error": cc["explicit"], "trotter_order": 2, "updates_per_step": upd,
            "parallelism": f"sites sharded x{ws} (contiguous even-aligned blocks)",
            "l2": "chain state (GBs) far larger than L2"}


def run_chain(args, cc, as_anchor=False):
    """C5: finite chain in Hastings form through the C-ABI sharded chain
    (qt_chain_*, qt_tebd_step_finite_sharded, csrc/chain.cu): contiguous
    even-aligned site blocks per rank, interior bonds on 8 concurrent worker
    contexts, the straddling tensors exchanged with ncclSend / ncclRecv of raw
    device buffers (the NCCL id broadcast over torch.distributed).  Strong
    scaling: the chain is fixed, value = Trotter steps/s of the whole chain
    from the max over ranks.  as_anchor: return the line instead of printing
    (the N=1 run's C5 point for a scaling curve)."""
    import torch

    from paper_2212_09782_b200 import _capi, model
    from paper_2212_09782_b200 import qrtebd as q
    from paper_2212_09782_b200.chain import DeviceChain, nccl_unique_id, partition
    from paper_2212_09782_b200.finite import chain_dims, random_chain_state

    if args.impl == "reference" and not as_anchor:
        return run_chain_reference(args, cc)
    ws, rank, local = (1, 0, 0) if as_anchor else dist_setup()
    import torch.distributed as dist_mod
    n, d, chi, scheme, explicit = cc["n"], cc["d"], cc["chi"], cc["scheme"], cc["explicit"]
    torch.cuda.set_device(local)
    ctx = _capi.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    dmma_peak = ctx.fp64_peak(0)
    start, end = partition(n, ws, rank)
    sites, bonds, keep = random_chain_state(ctx, n, d, chi, start, end)
    nid = None
    if ws > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist_mod.broadcast_object_list(obj, src=0)
        nid = obj[0]
    workers = max(0, int(os.environ.get("QT_CHAIN_STREAMS", "8")))
    chain = DeviceChain(ctx, n, sites, bonds, rank, ws, nccl_id=nid, workers=workers)
    del sites, bonds, keep
    layers = []
    for parity, dte in model.layer_structure(0.05, 2):
        layers.append((0 if parity == "even" else 1,
                       [ctx.tensor(model.make_gate(model.chain_bond_hamiltonian(d, 2.0, m, n), dte))
                        if start <= m + 1 and m < end else None for m in range(n - 1)]))
    pol = q.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=explicit)
    steps = 2 if as_anchor else args.steps
    warmup = 1 if as_anchor else (max(1, min(args.warmup, 2)) if args.steps <= 3 else args.warmup)
    for _ in range(warmup):
        chain.step(layers, scheme, pol)
    sampler = ClockSampler(local)
    sampler.start()
    barrier(ws)
    torch.cuda.synchronize()
    ctx.synchronize()
    launches0 = ctx.lib.qt_kernel_launches()
    step_ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        chain.step(layers, scheme, pol)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier(ws)
    clocks = sampler.stop()
    launches = ctx.lib.qt_kernel_launches() - launches0
    tot_ms = max_over_ranks(sum(step_ms), ws)
    ms_per_step = tot_ms / steps

    # ---------------- e2e: this rank's block of the chain (site tensors and
    # bond matrices) copied in from pinned host memory before and out after
    # every step, through the same C-ABI calls
    def state_views():
        return [chain.view("site", m) for m in range(start, end)] + [chain.view("bond", m) for m in range(start, end)]

    host_in = [torch.from_numpy(np.ascontiguousarray(v.numpy()).view(np.float64)).pin_memory() for v in state_views()]
    host_out = [torch.empty_like(t).pin_memory() for t in host_in]
    h2d = sum(t.numel() * 8 for t in host_in)
    lib = ctx.lib
    barrier(ws)
    ctx.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(steps):
        for t, hb in zip(state_views(), host_in):
            _capi.check(lib.qt_tensor_upload_async(t.h, _capi.C.cast(hb.data_ptr(), _capi.DP)))
        chain.step(layers, scheme, pol)
        for t, hb in zip(state_views(), host_out):
            _capi.check(lib.qt_tensor_download_async(t.h, _capi.C.cast(hb.data_ptr(), _capi.DP)))
    f1.record(stream)
    ctx.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), ws) / steps
    chis = chain_dims(n, d, chi)
    f_step = 0.0
    for parity, _ in layers:
        for m in range(parity, n - 1, 2):
            cn = chis[m + 1]
            eta = min(cn, chis[m] * d, d * chis[m + 2])
            f_step += flops_per_update(d, cn, eta, eta, explicit)  # uniform-chi estimate per bond
    upd_per_step = sum(len(range(p, n - 1, 2)) for p, _ in layers)
    line = {
        "metric": METRIC, "value": 1e3 / ms_per_step, "unit": "steps/s", "n_gpus": ws, "steps": steps,
        "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
        "config": chain_config_dict(cc, ws),
        "path": f"C-ABI qt_tebd_step_finite_sharded: {workers} worker contexts per rank, NCCL send/recv of the "
                "straddling site tensors" if ws > 1 else f"C-ABI qt_tebd_step_finite_sharded, {workers} worker contexts",
        "updates_per_s": upd_per_step * 1e3 / ms_per_step,
        "step_ms": [round(x, 3) for x in step_ms],
        "e2e": {"value": 1e3 / e2e_ms, "unit": "steps/s", "h2d_bytes_per_step": h2d * ws, "d2h_bytes_per_step": h2d * ws,
                "scope": "each rank's site tensors and bond matrices from pinned host memory in and out every step"},
        "roofline": {"bound": "tensor", "achieved": f_step / (ms_per_step * 1e-3) / 1e12, "peak": dmma_peak * ws,
                     "unit": "TFLOP/s", "frac": f_step / (ms_per_step * 1e-3) / 1e12 / (dmma_peak * ws),
                     "traffic": None, "scope": "whole chain step (all kernels), algorithmic flops / device time",
                     "flops_per_step": f_step, "complex_products": COMPLEX_3M_NOTE,
                     "frac_of_3m_peak": f_step / (ms_per_step * 1e-3) / 1e12 / (dmma_peak * ws * 4.0 / 3.0)},
        "gpu_launches": int(launches), "clocks": clocks,
    }
    chain.close()
    del layers
    ctx.close()
    if as_anchor:
        return line
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist_mod.destroy_process_group()
    return 0


def run_chain_reference(args, cc):
    """CPU reference arm for C5: the oracle's bond update timed on the host
    cores on a bounded sample (the chain's central chi x chi bonds); a step is
    extrapolated as (updates per step) x (mean central-bond update time), an
    upper bound since edge bonds are cheaper."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    n, d, chi = cc["n"], cc["d"], cc["chi"]
    upd = 2 * len(range(0, n - 1, 2)) + len(range(1, n - 1, 2))
    # the reference itself (oracle/_ref/ref_bench) on a central chi x chi bond
    # cell, when it is built: per-update time x updates per chain step
    cell = (f"C5 central bond d={d}, chi={chi}", d, chi, cc["scheme"], cc["explicit"], (0, 0.0))
    rb = reference_binary_rate(cell, budget_s=20.0, min_updates=3)
    if rb is not None:
        cell_rate, n_upd, secs, threads = rb
        t_upd = secs / n_upd
        rate = 1.0 / (upd * t_upd)
        line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s", "n_gpus": args.gpus,
                "steps": int(n_upd), "warmup": 1, "ms_per_step": 1e3 / rate, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
                "config": chain_config_dict(cc, int(os.environ.get("WORLD_SIZE", "1"))),
                "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": int(threads), "kind": "reference",
                                 "sample": f"{int(n_upd)} updates of a central chi={chi} bond cell by the reference's "
                                           f"own apply_gate (oracle/_ref/ref_bench, {secs:.1f} s), step = {upd} "
                                           "updates x mean update time (upper bound: edge bonds are cheaper)"},
                "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    from oracle import qrtebd_oracle as ref
    from paper_2212_09782_b200 import model
    rng = np.random.default_rng(0x51AB)
    bm = ref.random_right_isometry(rng, d, chi, chi)
    bn = ref.random_right_isometry(rng, d, chi, chi)
    xi = rng.standard_normal((chi, chi)) + 1j * rng.standard_normal((chi, chi))
    xi /= np.linalg.norm(xi)
    u = model.make_gate(model.chain_bond_hamiltonian(d, 2.0, n // 2, n), 0.05)
    pol = ref.TruncationPolicy(chi_max=chi, delta_chi_abs=0, delta_chi_rel=0.0, compute_explicit_error=cc["explicit"])
    ref.apply_gate_qr(xi, bm, bn, u, pol)
    k = max(1, args.steps)
    t0 = time.perf_counter()
    for _ in range(k):
        ref.apply_gate_qr(xi, bm, bn, u, pol)
    t_upd = (time.perf_counter() - t0) / k
    rate = 1.0 / (upd * t_upd)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s", "n_gpus": args.gpus,
            "steps": k, "warmup": 1, "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
            "config": chain_config_dict(cc, int(os.environ.get("WORLD_SIZE", "1"))),
            "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{k} central-bond updates (chi={chi}) of the NumPy/LAPACK oracle, step = "
                                       f"{upd} updates x mean update time (upper bound)"},
            "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def gemm_traffic(config):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of the
    dominant GEMM of this configuration, from the committed ncu --set full
    captures: north star = the X = theta Y0^H GEMM (5120 x 1024 x 5120,
    3M build, profiles/r02_final/gemm_x_raw.csv.gz); C2 = the 1280 x 256 x 1280
    projection (profiles/r01_ncu_full_summary.txt); None when no capture of
    that shape exists."""
    import csv
    import gzip
    import io
    here = os.path.dirname(os.path.abspath(__file__))
    if config == "north":
        path = os.path.join(here, "profiles", "r02_final", "gemm_x_raw.csv.gz")
        if not os.path.exists(path):
            return None
        rows = list(csv.reader(io.StringIO(gzip.open(path, "rt").read())))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for vals in rows[2:]:
            d = dict(zip(hdr, zip(vals, units)))
            if "zgemm_kernel<0, 1" not in d.get("Kernel Name", ("", ""))[0]:
                continue
            try:
                return sum(float(d[k][0].replace(",", "")) * scale[d[k][1]]
                           for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            except (KeyError, ValueError):
                return None
        return None
    if config != "c2":
        return None
    path = os.path.join(here, "profiles", "r01_ncu_full_summary.txt")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        lines = f.read().splitlines()
    cols = lines[0].split()
    for ln in lines[1:]:
        if ln.startswith("zgemm_c2.ncu-rep"):
            vals = ln.split()
            m = dict(zip(cols[2:], vals[-(len(cols) - 2):]))
            try:
                return (float(m["dram_read_MB"]) + float(m["dram_write_MB"])) * 1e6
            except (KeyError, ValueError):
                return None
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS) + sorted(CHAIN_CONFIGS),
                    help="default: north (N=1) / c5 sharded chain (N>1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scaling-anchor", action="store_true",
                    help="skip the 1-GPU C5 chain point appended to the default N=1 line")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--path", default="graph", choices=["graph", "value"],
                    help="graph: device-resident state, CUDA-graph step; value: C-ABI tebd_step (new handles)")
    args = ap.parse_args()
    if args.config is None:
        args.config = "north" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "c5"
    if args.config in CHAIN_CONFIGS:
        return run_chain(args, CHAIN_CONFIGS[args.config])
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    from paper_2212_09782_b200 import _capi, model
    from paper_2212_09782_b200 import qrtebd as q

    ws, rank, local = dist_setup()
    desc, d, chi, scheme, explicit, _ = cfg
    warmup = max(3, args.warmup)
    ctx = _capi.Context(local)
    lib = ctx.lib
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    dmma_peak = ctx.fp64_peak(0)

    sites_h, bonds_h = synthetic_state(d, chi)
    state0 = q.UniformMPS.from_numpy(ctx, d, sites_h, bonds_h)
    sched_h = [(p, model.make_gate(model.bond_hamiltonian(d, 2.0), dte)) for p, dte in model.layer_structure(0.05, 2)]
    sched = [(p, ctx.tensor(u)) for p, u in sched_h]
    pol = q.TruncationPolicy(**policy_kw(cfg))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > 126 MB L2

    # The fast path: state resident in HBM (qt_uniform_*), each step one CUDA
    # graph replay once the bond dimensions are stationary.  --path value
    # times the value-semantics C-ABI tebd_step instead (new handles per step).
    graph_path = args.path == "graph"
    # roofline evidence: CUDA-event pairs around the hot-path contraction GEMMs
    # (>= 5% of an update's flops: theta build, X = theta Y0^H, Hastings, the
    # explicit-error products).  The Householder block-reflector products --
    # including those applied to theta on a side stream behind the QR panels,
    # which share the SMs with both panel chains -- stay un-instrumented: their
    # event-bracketed durations measure the contention, not the kernel
    eta_cfg, kk_cfg = widths(cfg)
    prof_min_flops = 0.05 * flops_per_update(d, chi, eta_cfg, kk_cfg, explicit, cbe=(scheme == "qr_cbe"))
    if graph_path:
        # capture the step graphs with the GEMM event nodes in them (profiling
        # on); warm-up >= 4 so both buffer-parity graphs exist before timing
        warmup = max(warmup, 4)
        if not os.environ.get("QT_BENCH_NO_GRAPH_PROF"):
            _capi.check(lib.qt_profile_begin(ctx.h, prof_min_flops))
        dev = q.DeviceUniformMPS(state0, ctx)
        for _ in range(warmup):
            reps = dev.step(sched, scheme, pol)
    else:
        state = state0
        for _ in range(warmup):
            state, reps = q.tebd_step(state, sched, scheme, pol, ctx)
    assert all(r.report.chi_after == chi for r in reps)

    def one_step():
        nonlocal state
        if graph_path:
            return dev.step(sched, scheme, pol)
        state, r = q.tebd_step(state, sched, scheme, pol, ctx)
        return r

    # ---------------- timed region: device-resident state
    sampler = ClockSampler(local)
    sampler.start()
    barrier(ws)
    torch.cuda.synchronize()
    ctx.synchronize()
    launches0 = lib.qt_kernel_launches()
    _capi.check(lib.qt_profile_begin(ctx.h, prof_min_flops))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps, outside the event pair
        evs[k][0].record(stream)
        reps = one_step()
        evs[k][1].record(stream)
    ctx.synchronize()
    gf, gms, gl = (np.zeros(1), np.zeros(1), np.zeros(1, dtype=np.uint64))
    gfl, gmsl, gll = _capi.C.c_double(), _capi.C.c_double(), _capi.C.c_uint64()
    _capi.check(lib.qt_profile_end(ctx.h, _capi.C.byref(gfl), _capi.C.byref(gmsl), _capi.C.byref(gll)))
    launches = lib.qt_kernel_launches() - launches0
    torch.cuda.synchronize()
    barrier(ws)
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = max_over_ranks(sum(step_ms), ws)
    ms_per_step = tot_ms / args.steps
    value = ws * 1e3 / ms_per_step

    # ---------------- e2e: host (pinned) state in, host state out every step
    flat_in = [torch.from_numpy(np.ascontiguousarray(a).view(np.float64)).pin_memory() for a in sites_h + bonds_h]
    h2d = sum(t.numel() * 8 for t in flat_in)
    outs_pinned = [torch.empty_like(t).pin_memory() for t in flat_in]
    dev_in = [ctx.empty(a.shape) for a in sites_h + bonds_h]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    ctx.synchronize()
    e0.record(stream)
    for k in range(args.steps):
        if graph_path:
            # host state -> live device buffers, step, live buffers -> host
            views = [dev.view("site", m) for m in range(2)] + [dev.view("bond", m) for m in range(2)]
            for t, hbuf in zip(views, flat_in):
                _capi.check(lib.qt_tensor_upload_async(t.h, _capi.C.cast(hbuf.data_ptr(), _capi.DP)))
            dev.step(sched, scheme, pol)
            views = [dev.view("site", m) for m in range(2)] + [dev.view("bond", m) for m in range(2)]
            for t, hbuf in zip(views, outs_pinned):
                _capi.check(lib.qt_tensor_download_async(t.h, _capi.C.cast(hbuf.data_ptr(), _capi.DP)))
        else:
            for t, hbuf in zip(dev_in, flat_in):
                _capi.check(lib.qt_tensor_upload_async(t.h, _capi.C.cast(hbuf.data_ptr(), _capi.DP)))
            st_in = q.UniformMPS(d, dev_in[:2], dev_in[2:])
            st_out, _ = q.tebd_step(st_in, sched, scheme, pol, ctx)
            for t, hbuf in zip(st_out.site_tensors + st_out.bond_matrices, outs_pinned):
                _capi.check(lib.qt_tensor_download_async(t.h, _capi.C.cast(hbuf.data_ptr(), _capi.DP)))
    e1.record(stream)
    ctx.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), ws) / args.steps
    d2h = sum(t.numel() * 8 for t in outs_pinned)

    # ---------------- roofline: the whole step against the FP64 tensor pipe
    # achieved = SURVEY.md §8(d) algorithmic flops of one Trotter step (3
    # updates) / the device step time; the dominant DMMA GEMM kernel's own
    # rate (event-bracketed launches inside the timed graph) is a sub-field
    gemm_tf = gfl.value / (gmsl.value * 1e-3) / 1e12 if gmsl.value > 0 else 0.0
    eta, kk = widths(cfg)
    f_step = 3 * flops_per_update(d, chi, eta, kk, explicit, cbe=(scheme == "qr_cbe"))
    step_tf = f_step / (ms_per_step * 1e-3) / 1e12
    roofline = {
        "bound": "tensor", "achieved": step_tf, "peak": dmma_peak, "unit": "TFLOP/s",
        "frac": step_tf / dmma_peak if dmma_peak else None, "traffic": gemm_traffic(args.config),
        "scope": "whole Trotter step: SURVEY.md §8(d) algorithmic flops of 3 updates / device step time "
                 "(QR panels, block reflectors, permutes and GEMMs all inside the denominator)",
        "flops_per_step": f_step,
        "complex_products": COMPLEX_3M_NOTE,
        "peak_3m": dmma_peak * 4.0 / 3.0 if dmma_peak else None,
        "frac_of_3m_peak": step_tf / (dmma_peak * 4.0 / 3.0) if dmma_peak else None,
        "peak_source": "FP64 DMMA microbenchmark (csrc/probe.cu, mma.sync m8n8k4 f64 -> DMMA.8x8x4) measured in "
                       "this run; MEASURED_PEAKS.json has no FP64 figure",
        "traffic_note": "dram bytes (read + write) per launch of the dominant GEMM (north star: X = theta "
                        "Y0^H, 5120 x 1024 x 5120; compulsory A+B+C = 587 MB, so ~2x re-reads of theta at 178 flop/B -- compute-bound) from the committed ncu --set "
                        "full capture (profiles/r02/), null if none",
        "dominant_kernel": {
            "kernel": "zgemm_kernel (mma.sync m8n8k4 f64 -> DMMA, TMA-staged, mbarrier ring)",
            "achieved": gemm_tf, "frac": gemm_tf / dmma_peak if dmma_peak else None,
            "frac_of_3m_peak": gemm_tf / (dmma_peak * 4.0 / 3.0) if dmma_peak else None,
            "share_of_step": (gmsl.value / args.steps) / (sum(step_ms) / args.steps),
            "launches_per_step": int(gll.value) / args.steps,
            "bracketed": f"contraction launches >= {prof_min_flops:.3g} flops (theta build, X = theta Y0^H, "
                         "Hastings, explicit-error products); the QR pair's block-reflector products are not "
                         "bracketed"},
    }

    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": ws, "steps": args.steps, "warmup": warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128", "data": "synthetic",
        "config": config_dict(cfg, ws),
        "path": ("device-resident state, one CUDA graph replay per step (qt_uniform_step)"
                 if graph_path else "C-ABI qt_tebd_step_uniform, new handles per step"),
        "updates_per_s": 3 * value,
        "step_ms": [round(x, 3) for x in step_ms],
        "roofline": roofline,
        "e2e": {"value": ws * 1e3 / e2e_ms, "unit": "steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        refbin = reference_binary_rate(cfg, budget_s=args.cpu_budget)
        if refbin is not None:
            rate, n, dt, thr = refbin
            line["cpu_baseline"] = {"value": rate, "unit": "steps/s", "cores": thr, "kind": "reference",
                                    "sample": f"{n} bond updates ({n / 3:.2f} Trotter steps, {dt:.1f} s) of the "
                                              "reference itself (proj/src compiled in place on the Eigen-3.4-subset "
                                              "shim over OpenBLAS LAPACK, oracle/_ref/ref_bench) on the same config "
                                              f"and state, {thr} BLAS threads; steps/s = updates/3 / time",
                                    "host": host_info()}
        else:
            rate, n, dt = cpu_reference_rate(cfg, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {"value": rate, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"{n} bond updates ({n / 3:.2f} Trotter steps, {dt:.1f} s) of the "
                                              f"NumPy/LAPACK oracle port on the same config and state, OpenBLAS "
                                              f"threads = {os.cpu_count()}; steps/s = updates/3 / time",
                                    "host": host_info()}
        if chi <= 256:
            # the reference's SVD-TEBD comparator (gates.cpp:312-322) on the
            # same cell and truncation, timed beside it
            rate_s, n_s, dt_s = cpu_reference_rate(cfg, budget_s=max(1.0, args.cpu_budget / 3), scheme="svd")
            line["cpu_baseline_svd"] = {"value": rate_s, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                                        "sample": f"{n_s} updates ({dt_s:.1f} s) of the oracle's SVD-TEBD update "
                                                  "(zgesdd of theta) on the same state and gate schedule"}
    if graph_path:
        dev.close()
    ctx.close()
    if rank == 0 and ws == 1 and not args.no_scaling_anchor:
        # the N=1 point of the scaling curve: `bench.py --gpus N` (N > 1)
        # runs the C5 chain sharded over N ranks; its 1-GPU value, measured
        # here after the headline's timed region
        a = run_chain(args, CHAIN_CONFIGS["c5"], as_anchor=True)
        line["scaling_anchor"] = {"config": a["config"]["workload"], "n_gpus": 1, "value": a["value"],
                                  "unit": a["unit"], "ms_per_step": a["ms_per_step"], "steps": a["steps"],
                                  "roofline_frac": a["roofline"]["frac"], "path": a["path"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
