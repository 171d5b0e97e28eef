"""B200 benchmark: AES-128 encrypt GB/s of plaintext (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one pass of the hot path over one batch: encrypt every block of
the configured workload once (shared-IV CBC over 16-byte messages, i.e.
C_i = AES_K(P_i ^ IV), the reference's mode).

* ``value``   -- whole-job plaintext GB/s, inputs resident in HBM, CUDA events
                 on the launching stream, max over ranks.  ``wall_span``
                 beside it: host barrier -> last rank's completion.
* ``e2e``     -- the same metric through the public host-buffer API
                 (``backend_cuda.encrypt_shared_iv`` -> C ABI
                 ``gaes_encrypt_shared_iv``) with pinned host input/output:
                 H2D + kernel + D2H inside the timed region every step.
* ``roofline``-- binding roofline of the dominant kernel (shared-memory
                 table lookups, 144 per block + 16 texture S-box fetches)
                 plus the HBM roofline (32 algorithmic bytes per block).
* ``cpu_baseline`` -- the reference's own stock CPU path on the host cores,
                 rank 0 at N=1, on a bounded sample of the same workload:
                 ``parallel._run_chunks(backend.cbc_encrypt,
                 aes_cbc._encrypt_tables(key), P, IVSet.shared(iv).rows(n),
                 out, plan(n, W).chunks)`` from the unchanged package in
                 baseline/_ref (parallel.py:66-75, aes_cbc.py:333-336), and
                 the same for decrypt.  Where baseline/_ref is absent the
                 reference's own compiled kernel from oracle/_ref runs over the
                 same plan.  This leg and ``--impl reference`` are the only
                 places bench.py touches oracle/; the GPU arm verifies against
                 golden digests, an independent formulation and round trips.

Workloads (BASELINE.json configs; seeded synthetic data -- configs 1/2 use the
reference bench's own recipe so the output is checked against the golden
ciphertext digests, configs 3/4/5 are generated on the device in 2^22-block
chunks seeded by their global index, so the bytes do not depend on N):
  1: 2^16 uniform blocks per GPU (weak)     2: 2^24 uniform blocks per GPU (weak)
  3: 2^28 sensor-stream blocks, sharded (strong; the default: the first config
     the 1/2/4/8-B200 metric is quoted on)
  4: 2^26 Zipf(1.1) uint64 blocks, sharded  5: 1024 keys x 2^20 blocks, keys sharded
``--impl reference`` times the reference CPU path instead (rank 0 only), on
the same ``config`` dict.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BYTES_PER_BLOCK = 16
LOOKUPS_PER_BLOCK = 160  # 9 rounds x 16 T-table lookups + 16 S-box lookups
T_LOOKUPS_PER_BLOCK = 144  # the T-table rounds 1-9 (shared memory)
# BASELINE.json's metric, verbatim (the roofline fraction is the `roofline` object)
METRIC = "AES-128 encrypt GB/s of plaintext (1/2/4/8 B200) and % of roofline"
HBM_BYTES_PER_BLOCK = 32  # 16 read + 16 written (shared IV folded into the key)
SEED = 2016  # bench.py:49 default seed in the reference
DEFAULT_CONFIG = 3
GEN_CHUNK_BLOCKS = 1 << 22  # device generation granularity (shard-invariant bytes)
PIECES = 8  # strong-scaled workloads are digested in 8 equal pieces (N = 1, 2, 4, 8 own whole pieces)
CPU_SAMPLE_CAP = 1 << 24  # CPU arms: at most 2^24 blocks (256 MiB) per timed sample


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-digests", action="store_true", help="skip the per-piece ciphertext digests")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline budget")
    ap.add_argument("--cpu-sample-cap", type=int, default=CPU_SAMPLE_CAP, help="CPU arms: blocks per sample (max)")
    ap.add_argument("--variant", type=int, default=0)
    return ap.parse_args(argv)


WORKLOADS = {
    1: dict(name="cfg1: 2^16 uniform 16-B blocks per GPU, one key, shared IV", blocks=1 << 16, scaling="weak"),
    2: dict(name="cfg2: 2^24 uniform 16-B blocks (256 MiB) per GPU, one key, shared IV", blocks=1 << 24,
            scaling="weak"),
    3: dict(name="cfg3: 2^28 sensor-stream blocks (4 GiB) sharded over GPUs, one key", blocks=1 << 28,
            scaling="strong"),
    4: dict(name="cfg4: 2^26 Zipf(1.1) uint64 column blocks (1 GiB) sharded, one key", blocks=1 << 26,
            scaling="strong"),
    5: dict(name="cfg5: 1024 keys x 2^20 blocks (16 GiB), keys sharded, GPU key schedule", blocks=1 << 30,
            scaling="strong", keys=1024),
}


# ----------------------------------------------------------------------------- workload geometry

def plan_chunks(n: int, workers: int) -> list:
    """Balanced contiguous ranges, sizes within one (parallel.py:37-50; the
    same rule as paper_1506_08503_b200.shard.plan -- restated here so the
    reference arm never loads this repo's package)."""
    k = min(workers, n)
    if k <= 0:
        return []
    q, r = divmod(n, k)
    edges = [i * q + min(i, r) for i in range(k + 1)]
    return list(zip(edges[:-1], edges[1:]))


def _slice(n: int, rank: int, world: int) -> tuple:
    chunks = plan_chunks(n, world)
    return chunks[rank] if rank < len(chunks) else (n, n)


def rank_range(cfg: int, rank: int, world: int, blocks: int | None = None) -> tuple:
    """Global blocks [lo, hi) this rank encrypts.  Weak configs: the whole
    workload on every rank; strong: the reference's plan (parallel.py:37-50)
    over blocks, or over keys for config 5."""
    w = WORKLOADS[cfg]
    total = blocks or w["blocks"]
    if w["scaling"] == "weak":
        return 0, total
    if cfg == 5:
        bpk = total // w["keys"]
        k_lo, k_hi = _slice(w["keys"], rank, world)
        return k_lo * bpk, k_hi * bpk
    return _slice(total, rank, world)


def total_blocks(cfg: int, world: int) -> int:
    w = WORKLOADS[cfg]
    return w["blocks"] * world if w["scaling"] == "weak" else w["blocks"]


def pieces(cfg: int, blocks: int | None = None) -> list:
    """The PIECES equal ranges a strong workload is digested in (key-aligned
    for config 5)."""
    w = WORKLOADS[cfg]
    total = blocks or w["blocks"]
    if cfg == 5:
        bpk = total // w["keys"]
        return [(a * bpk, b * bpk) for a, b in plan_chunks(w["keys"], PIECES)]
    return plan_chunks(total, PIECES)


def l2_policy(cfg: int, world: int) -> str:
    lo, hi = rank_range(cfg, 0, world)
    return ("ring of K cold copies of the batch (one L2 flush before the region), K steps as one CUDA graph"
            if (hi - lo) * 32 < (256 << 20) else "inputs larger than L2 (no flush)")


def workload_params(cfg: int, blocks: int | None = None) -> dict:
    """Key, IV and the generator parameters of a config -- pure numpy, so the
    GPU arm and the reference arm describe (and draw) the same workload."""
    w = WORKLOADS[cfg]
    rng = np.random.default_rng(SEED)
    key, iv = rng.bytes(16), rng.bytes(16)  # bench.py:124-125 draw order
    prm = {"rng": rng, "key": key, "iv": iv,
           "meta": {"seed": SEED, "key": key.hex(), "iv": iv.hex()}}
    if cfg in (1, 2):
        prm["meta"]["recipe"] = "numpy default_rng(2016): key, iv, uniform bytes (reference bench.py:124-126)"
    elif cfg == 3:
        f = rng.uniform(0.001, 0.1, 3)
        a = rng.uniform(1000, 8000, 3)
        phi = rng.uniform(0, 2 * np.pi, 3)
        prm.update(f=f, a=a, phi=phi)
        prm["meta"].update(freqs=f.tolist(), amps=a.tolist(), phases=phi.tolist(), sigma=200,
                           block="8 little-endian int16 samples")
    elif cfg == 4:
        nvals = 10 ** 6
        vals = np.unique(rng.integers(0, 2 ** 64, int(nvals * 1.05), dtype=np.uint64))
        vals = rng.permutation(vals)[:nvals]
        ranks_w = np.arange(1, nvals + 1, dtype=np.float64) ** -1.1
        prm.update(vals=vals, cdf=np.cumsum(ranks_w) / ranks_w.sum())
        prm["meta"].update(zipf_s=1.1, distinct=nvals, block="uint64 LE + 8 zero bytes")
    else:
        keys = rng.integers(0, 256, (w["keys"], 16), dtype=np.uint8)
        ivs = rng.integers(0, 256, (w["keys"], 16), dtype=np.uint8)
        prm.update(keys=keys, ivs=ivs, bpk=(blocks or w["blocks"]) // w["keys"])
        prm["meta"].update(keys=w["keys"], blocks_per_key=prm["bpk"], iv="one shared IV per key")
    return prm


def config_dict(cfg: int, world: int) -> dict:
    """The `config` object -- identical in both arms (driver's same_config)."""
    w = WORKLOADS[cfg]
    lo, hi = rank_range(cfg, 0, world)
    shard = "contiguous key shards" if cfg == 5 else "contiguous block shards"
    return {"workload": w["name"], "total_blocks": total_blocks(cfg, world), "blocks_per_gpu": hi - lo,
            "scaling": w["scaling"], "parallelism": f"dp{world} ({shard}, no collective)",
            "l2": l2_policy(cfg, world), **workload_params(cfg)["meta"]}


# ----------------------------------------------------------------------------- inputs

def _chunked(lo: int, hi: int, fill):
    """fill(chunk_index, chunk_lo, a, b) for every GEN_CHUNK_BLOCKS chunk that
    overlaps [lo, hi); [a, b) is the overlap in global blocks."""
    C = GEN_CHUNK_BLOCKS
    for c in range(lo // C, (hi + C - 1) // C):
        a, b = max(lo, c * C), min(hi, (c + 1) * C)
        if a < b:
            fill(c, c * C, a, b)


def make_inputs(cfg: int, rank: int, world: int, device, blocks: int | None = None):
    """Seeded synthetic plaintext for this rank, generated on the device.

    Configs 3/4/5 draw each 2^22-block chunk from a generator seeded by the
    chunk's global index (the full chunk is drawn and the rank keeps its
    overlap), so a block's bytes do not depend on the rank count.  ``blocks``
    overrides the workload size (tests use small instances of the same
    generators)."""
    import torch

    prm = workload_params(cfg, blocks)
    rng, key, iv = prm["rng"], prm["key"], prm["iv"]
    lo, hi = rank_range(cfg, rank, world, blocks)
    n = hi - lo
    out = dict(key=key, iv=iv, lo=lo, hi=hi, meta=prm["meta"])
    C = GEN_CHUNK_BLOCKS

    def gen(c):
        g = torch.Generator(device=device)
        g.manual_seed(SEED * 1000 + cfg * 100000 + c)
        return g

    if cfg in (1, 2):
        # the reference bench recipe (bench.py:124-126): the same bytes the
        # golden digests in tests/golden/golden.json were computed from
        out["p"] = torch.from_numpy(rng.integers(0, 256, (n, 16), dtype=np.uint8)).to(device)
        out["meta"] = dict(prm["meta"], golden="tests/golden/golden.json digests[%d]" % n)
        return out
    p = torch.empty((n, 16), dtype=torch.uint8, device=device)
    if cfg == 3:
        f, a, phi = prm["f"], prm["a"], prm["phi"]
        samples = p.view(torch.int16).view(-1)  # 8 LE int16 per block

        def fill(c, c0, s, e):
            noise = torch.randn(8 * min(C, (blocks or WORKLOADS[3]["blocks"]) - c0), dtype=torch.float64,
                                device=device, generator=gen(c))[8 * (s - c0):8 * (e - c0)]
            t = torch.arange(8 * s, 8 * e, dtype=torch.float64, device=device)
            x = noise.mul_(200.0)
            for k in range(3):
                x += a[k] * torch.sin(2 * np.pi * f[k] * t + phi[k])
            samples[8 * (s - lo):8 * (e - lo)] = torch.clamp(torch.round(x), -32768, 32767).to(torch.int16)
        _chunked(lo, hi, fill)
    elif cfg == 4:
        cdf = torch.from_numpy(prm["cdf"]).to(device)
        vals = torch.from_numpy(prm["vals"].view(np.int64)).to(device)

        def fill(c, c0, s, e):
            u = torch.rand(min(C, (blocks or WORKLOADS[4]["blocks"]) - c0), dtype=torch.float64, device=device,
                           generator=gen(c))[s - c0:e - c0]
            r = torch.searchsorted(cdf, u).clamp_(max=vals.numel() - 1)
            p[s - lo:e - lo, :8] = vals[r].view(torch.uint8).view(e - s, 8)
            p[s - lo:e - lo, 8:] = 0
        _chunked(lo, hi, fill)
    else:  # cfg 5: many keys; this rank's keys and their blocks
        bpk = prm["bpk"]
        total = bpk * WORKLOADS[5]["keys"]

        def fill(c, c0, s, e):
            x = torch.randint(0, 256, (min(C, total - c0), 16), dtype=torch.uint8, device=device, generator=gen(c))
            p[s - lo:e - lo] = x[s - c0:e - c0]
        _chunked(lo, hi, fill)
        out.update(keys=prm["keys"][lo // bpk:hi // bpk], ivs=prm["ivs"][lo // bpk:hi // bpk], bpk=bpk)
    out["p"] = p
    return out


def cpu_sample(cfg: int, n: int) -> tuple:
    """A bounded host sample of the workload for the CPU arms: the first n
    blocks' worth of the same generator recipe (numpy draws; the device's
    noise / uniform streams are not reproduced byte for byte -- AES cost does
    not depend on the bytes).  Returns (P u8[n,16], [(key, iv, lo, hi), ...])."""
    prm = workload_params(cfg)
    rng, key, iv = prm["rng"], prm["key"], prm["iv"]
    if cfg in (1, 2):
        return rng.integers(0, 256, (n, 16), dtype=np.uint8), [(key, iv, 0, n)]
    if cfg == 3:
        p = np.empty((n, 16), np.uint8)
        s = p.view(np.int16).reshape(-1)
        step = 1 << 24
        for t0 in range(0, s.size, step):
            t = np.arange(t0, min(s.size, t0 + step), dtype=np.float64)
            x = 200.0 * rng.standard_normal(t.size)
            for k in range(3):
                x += prm["a"][k] * np.sin(2 * np.pi * prm["f"][k] * t + prm["phi"][k])
            s[t0:t0 + t.size] = np.clip(np.rint(x), -32768, 32767).astype("<i2")
        return p, [(key, iv, 0, n)]
    if cfg == 4:
        r = np.searchsorted(prm["cdf"], rng.random(n)).clip(max=prm["vals"].size - 1)
        p = np.zeros((n, 16), np.uint8)
        p[:, :8] = prm["vals"][r].view(np.uint8).reshape(n, 8)
        return p, [(key, iv, 0, n)]
    # cfg 5: the first keys, each with the workload's 2^20 blocks (fewer for
    # a sample below one key's share) -- the per-key call the reference makes
    per_key = (1 << 30) // WORKLOADS[5]["keys"]
    nk = max(1, min(WORKLOADS[5]["keys"], n // per_key))
    per = max(1, n // nk)
    p = rng.integers(0, 256, (nk * per, 16), dtype=np.uint8)
    return p, [(prm["keys"][i].tobytes(), prm["ivs"][i].tobytes(), i * per, (i + 1) * per) for i in range(nk)]


# ----------------------------------------------------------------------------- clocks

def _smi_index(local: int) -> int:
    """nvidia-smi index of CUDA device `local` (CUDA_VISIBLE_DEVICES-aware)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    parts = [v.strip() for v in vis.split(",") if v.strip()]
    if parts and local < len(parts) and parts[local].isdigit():
        return int(parts[local])
    return local


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def wait_first(self, timeout: float = 5.0):
        t0 = time.time()
        while self.proc is not None and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.01)

    def mark(self) -> int:
        return len(self.rows)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.reader.join(timeout=2)

    def summary(self, start: int = 0):
        rows = self.rows[start:] or self.rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = [x for x in (num(r[1]) for r in rows) if x is not None]
        smax = [x for x in (num(r[2]) for r in rows) if x is not None]
        pw = [x for x in (num(r[3]) for r in rows) if x is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------- CPU reference

def _ref_package():
    """The unchanged reference package installed in baseline/_ref (its
    compiled backend), or None."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "gaes")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import gaes
        from gaes import aes_cbc, parallel  # noqa: F401
    except Exception:  # pragma: no cover - informational only
        return None
    if "compiled" not in gaes.backend.available():
        return None
    return gaes


def _ref_kernel():
    """The reference's own compiled kernel (oracle/_ref, from _kernel.pyx)."""
    sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
    try:
        import _kernel  # type: ignore
        return _kernel
    except ImportError:
        return None
    finally:
        sys.path.pop(0)


class ReferenceCPU:
    """The reference's CPU path on a host sample, run the way its own data
    parallel layer runs it: parallel._run_chunks(kernel, tables, P,
    IVSet.shared(iv).rows(n), out, plan(n, W).chunks) (parallel.py:66-75,
    aes_cbc.py:333-342).  ``kind``: "reference" when baseline/_ref (the
    unchanged package, compiled backend) or oracle/_ref (its _kernel.pyx
    compiled from the sources) runs; "port" for the C oracle."""

    def __init__(self, cfg: int, n: int, threads: int):
        self.threads = threads
        self.p, self.segs = cpu_sample(cfg, n)
        self.n = self.p.shape[0]
        gaes = _ref_package()
        self.out = np.empty_like(self.p)
        self.back = np.empty_like(self.p)
        if gaes is not None:
            from gaes import aes_cbc, parallel
            gaes.backend.select("compiled")
            self.kind, self.source = "reference", "baseline/_ref (unchanged gaes package, compiled backend)"
            self._enc, self._dec = gaes.backend.cbc_encrypt, gaes.backend.cbc_decrypt
            self._run_chunks = parallel._run_chunks
            self._plan = lambda m: parallel.plan(m, threads).chunks
            self._tables = lambda k: (aes_cbc._encrypt_tables(k), aes_cbc._decrypt_tables(k))
            self._rows = lambda iv, m: aes_cbc.IVSet.shared(iv).rows(m)
        else:
            from oracle import oracle
            kern = _ref_kernel()
            if kern is not None:
                self.kind, self.source = "reference", "oracle/_ref (reference _kernel.pyx compiled from its sources)"
                self._enc, self._dec = kern.cbc_encrypt, kern.cbc_decrypt
            else:
                self.kind, self.source = "port", "oracle/gaes_oracle.c"
                self._enc = lambda *a: oracle.cbc_encrypt(*a)
                self._dec = lambda *a: oracle.cbc_decrypt(*a)
            self._run_chunks = _run_chunks_local
            self._plan = lambda m: oracle.plan(m, threads)
            self._tables = lambda k: (oracle.encrypt_tables(k), oracle.decrypt_tables(k))
            self._rows = lambda iv, m: np.tile(np.frombuffer(iv, np.uint8), (m, 1))
        # per key segment: tables, IV rows, chunk plan (prepared once, as the
        # reference's encrypt_batch_parallel does before its kernel fan-out)
        self.jobs = []
        for key, iv, lo, hi in self.segs:
            enc_t, dec_t = self._tables(key)
            self.jobs.append((lo, hi, enc_t, dec_t, self._rows(iv, hi - lo), self._plan(hi - lo)))

    def encrypt(self):
        for lo, hi, enc_t, _, rows, chunks in self.jobs:
            self._run_chunks(self._enc, enc_t, self.p[lo:hi], rows, self.out[lo:hi], chunks)

    def decrypt(self):
        for lo, hi, _, dec_t, rows, chunks in self.jobs:
            self._run_chunks(self._dec, dec_t, self.out[lo:hi], rows, self.back[lo:hi], chunks)

    def timed(self, fn, reps: int, warm: int) -> list:
        for _ in range(warm):
            fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return ts

    def check(self):
        """The sample's ciphertext agrees with the oracle and decrypts back."""
        from oracle import oracle
        lo, hi, *_ = self.jobs[0]
        key, iv = self.segs[0][0], self.segs[0][1]
        m = min(256, hi - lo)
        want = oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (m, 1)), self.p[lo:lo + m])
        assert np.array_equal(self.out[lo:lo + m], want), "CPU reference disagrees with the oracle"


def _run_chunks_local(kernel, tables, data, iv_rows, out, chunks):
    """parallel._run_chunks (parallel.py:66-75) for the fallbacks."""
    if len(chunks) <= 1:
        kernel(data, iv_rows, *tables, out)
        return
    with ThreadPoolExecutor(max_workers=len(chunks)) as pool:
        for f in [pool.submit(kernel, data[lo:hi], iv_rows[lo:hi], *tables, out[lo:hi]) for lo, hi in chunks]:
            f.result()


def _cpu_rate_probe(cfg: int, threads: int, n: int = 1 << 16) -> float:
    """Blocks/s of the reference CPU path on this host (a 2^16-block probe)."""
    r = ReferenceCPU(cfg, n, threads)
    return r.n / min(r.timed(r.encrypt, 2, 1))


def cpu_baseline(cfg: int, budget_s: float):
    threads = os.cpu_count() or 1
    rate = _cpu_rate_probe(cfg, threads)
    n = int(min(CPU_SAMPLE_CAP, max(1 << 16, rate * budget_s / 8)))
    r = ReferenceCPU(cfg, n, threads)
    # ~budget_s of CPU work in all: as many encrypt repetitions as ~60 % of
    # the budget holds (4..40), half as many decrypt ones
    t_one = r.timed(r.encrypt, 1, 1)[0]
    reps = int(max(4, min(40, 0.6 * budget_s / max(t_one, 1e-6))))
    enc = r.timed(r.encrypt, reps, 0)
    dec = r.timed(r.decrypt, max(2, reps // 2), 0)
    r.check()
    assert np.array_equal(r.back, r.p), "CPU reference round trip failed"
    one = ReferenceCPU(cfg, 1 << 18, 1)
    t1 = one.timed(one.encrypt, 1, 0)
    try:
        import psutil
        physical = psutil.cpu_count(logical=False)
    except Exception:  # pragma: no cover
        physical = None
    gbs = lambda ts, m: round(m * BYTES_PER_BLOCK / statistics.median(ts) / 1e9, 4)  # noqa: E731
    return {"value": gbs(enc, r.n), "unit": "GB/s", "cores": threads, "kind": r.kind,
            "sample": (f"{r.n} blocks of the workload (first blocks of its generator recipe, numpy draws), median of "
                       f"{len(enc)} reps, {threads} threads over parallel.plan chunks, parallel._run_chunks; "
                       f"{sum(enc) + sum(dec):.1f} s wall on {threads} threads"),
            "source": r.source,
            "decrypt": {"value": gbs(dec, r.n), "unit": "GB/s", "cores": threads,
                        "sample": f"the same {r.n} blocks, median of {len(dec)} reps (cbc_decrypt, _decrypt_tables)"},
            "single_thread": {"value": gbs(t1, one.n), "unit": "GB/s", "sample": f"{one.n} blocks, 1 thread"},
            "logical_cpus": threads, "physical_cores": physical}


def reference_api_e2e(key: bytes, iv: bytes, n: int = 1 << 16):
    """the reference's own public entry point end to end at
    config 1 -- gaes.encrypt_batch_parallel(key, IVSet.shared(iv), batch) on
    the unchanged package from baseline/_ref -- with its compiled backend on
    all host threads, and the same call with this repo's cuda backend
    registered (drop-in; one worker).  Batch construction is outside the
    timing.  None when baseline/_ref is absent."""
    gaes = _ref_package()
    if gaes is None:
        return None
    from gaes import parallel

    from paper_1506_08503_b200 import plugin
    rng = np.random.default_rng(SEED)
    data = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    batch = gaes.MessageBatch(data=data, original_lens=(16,) * n)
    ivs = gaes.IVSet.shared(iv)
    threads = os.cpu_count() or 1
    prev = gaes.backend.name()

    def timed(workers):
        parallel.encrypt_batch_parallel(key, ivs, batch, workers)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            out = parallel.encrypt_batch_parallel(key, ivs, batch, workers)
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), out

    try:
        gaes.backend.select("compiled")
        t_ref, c_ref = timed(threads)
        plugin.register(gaes_module=gaes, select=True)
        t_gpu, c_gpu = timed(1)
    finally:
        gaes.backend.select(prev)
    return {"api": "gaes.encrypt_batch_parallel(key, IVSet.shared(iv), batch) -- config 1, 65536 x 16 B",
            "reference": {"backend": "compiled", "workers": threads, "ms": round(t_ref * 1e3, 3),
                          "gbs": round(n * 16 / t_ref / 1e9, 4)},
            "cuda_backend": {"workers": 1, "ms": round(t_gpu * 1e3, 3), "gbs": round(n * 16 / t_gpu / 1e9, 4)},
            "identical_bytes": bool(np.array_equal(c_ref, c_gpu))}


def _openssl_worker(args):
    key, iv, n, budget_s, seed = args
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    p = np.random.default_rng(seed).integers(0, 256, (n, 16), dtype=np.uint8)
    x = (p ^ np.frombuffer(iv, np.uint8)).tobytes()
    enc = Cipher(algorithms.AES(key), modes.ECB()).encryptor()
    enc.update(x)
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < budget_s:
        enc.update(x)
        reps += 1
    return n * 16 * reps / (time.perf_counter() - t0)


def openssl_rate(key: bytes, iv: bytes, budget_s: float = 2.0):
    """OpenSSL AES-128-ECB of P ^ IV (AES-NI) on all host cores, one process
    per core: the paper's own comparand, reported beside
    cpu_baseline.  Returns None if the `cryptography` package is missing."""
    try:
        import cryptography  # noqa: F401
        from concurrent.futures import ProcessPoolExecutor
    except ImportError:
        return None
    procs = os.cpu_count() or 1
    n = 1 << 18
    import multiprocessing as mp
    with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn")) as pool:
        rates = list(pool.map(_openssl_worker, [(key, iv, n, budget_s, SEED + 2 + i) for i in range(procs)]))
    return {"value": round(sum(rates) / 1e9, 3), "unit": "GB/s", "cores": procs,
            "sample": f"{procs} processes x {n} blocks, AES-128-ECB of P^IV via OpenSSL (cryptography), "
                      f"{budget_s:.0f} s each"}


def openssl_sample_check(inp, p, out, cfg: int, n_sample: int = 1 << 16):
    """(ok, blocks checked) for a seeded random sample of this rank's blocks
    against OpenSSL AES-128-ECB of P ^ IV (per key for config 5), or None if
    the `cryptography` package is missing."""
    try:
        from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    except ImportError:
        return None
    import torch
    n = p.shape[0]
    rows = np.sort(np.random.default_rng(SEED + 7).choice(n, min(n, n_sample), replace=False))
    idx = torch.from_numpy(rows).to(p.device)
    ph, ch = p[idx].cpu().numpy(), out[idx].cpu().numpy()
    if cfg == 5:
        kidx = rows // inp["bpk"]
        ok = True
        for k in np.unique(kidx):
            sel = kidx == k
            enc = Cipher(algorithms.AES(inp["keys"][k].tobytes()), modes.ECB()).encryptor()
            want = np.frombuffer(enc.update((ph[sel] ^ inp["ivs"][k]).tobytes()), np.uint8).reshape(-1, 16)
            ok &= bool(np.array_equal(want, ch[sel]))
        return ok, int(rows.size)
    enc = Cipher(algorithms.AES(inp["key"]), modes.ECB()).encryptor()
    want = np.frombuffer(enc.update((ph ^ np.frombuffer(inp["iv"], np.uint8)).tobytes()), np.uint8).reshape(-1, 16)
    return bool(np.array_equal(want, ch)), int(rows.size)


def run_reference_impl(args):
    """--impl reference: the reference's stock CPU path, rank 0 only, on the
    same config / metric / unit as our arm; each step encrypts a bounded
    sample of the workload (at most 2^24 blocks)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    threads = os.cpu_count() or 1
    rate = _cpu_rate_probe(args.config, threads, min(1 << 16, args.cpu_sample_cap))
    budget_per_step = min(5.0, 150.0 / max(1, args.steps + args.warmup))
    n = int(min(args.cpu_sample_cap, max(min(1 << 16, args.cpu_sample_cap), rate * budget_per_step)))
    r = ReferenceCPU(args.config, n, threads)
    times = r.timed(r.encrypt, args.steps, args.warmup)
    r.check()
    dec = r.timed(r.decrypt, max(1, min(3, args.steps)), 0)
    assert np.array_equal(r.back, r.p), "CPU reference round trip failed"
    total = sum(times)
    value = r.n * args.steps * BYTES_PER_BLOCK / total / 1e9
    sample = (f"{r.n} blocks of the workload per step (first blocks of its generator recipe, numpy draws), "
              f"{threads} host threads, parallel._run_chunks over parallel.plan chunks")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": WORKLOADS[args.config]["scaling"], "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded, the workload's generator recipe on the host)",
        "config": config_dict(args.config, world),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": r.kind, "sample": sample,
                         "source": r.source},
        "decrypt": {"value": r.n * len(dec) * BYTES_PER_BLOCK / sum(dec) / 1e9, "unit": "GB/s",
                    "sample": f"the same {r.n} blocks, cbc_decrypt with _decrypt_tables"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- ours

def host_api_legs(args, inp, p, n, iv, rk, ch, world, rank, reduce_dev, launched):
    """`e2e` (the public host-buffer API with pinned buffers, H2D + kernel +
    D2H inside every timed step) and `e2e_dropin` (the reference's 7-argument
    backend call with pageable numpy buffers).  Returns (e2e, dropin, ok)."""
    import torch
    import torch.distributed as dist

    from paper_1506_08503_b200 import backend_cuda
    from paper_1506_08503_b200.shard import max_over_ranks

    cfg = args.config
    job_blocks = n * world if WORKLOADS[cfg]["scaling"] == "weak" else total_blocks(cfg, world)
    ok = True
    e2e = None
    if not args.no_e2e:
        h_in = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        h_in.copy_(p)
        hi, ho = h_in.numpy(), h_out.numpy()
        if cfg == 5:
            # keys + data from pinned host memory through the host many-key
            # entry point (key schedule on the GPU inside the step)
            call = lambda: backend_cuda.many_key_encrypt(hi, inp["keys"], inp["ivs"], out=ho)  # noqa: E731
            api = ("backend_cuda.many_key_encrypt -> gaes_many_key_encrypt (pinned host buffers, GPU key "
                   "schedule per step)")
            h2d = int(n * 16 + inp["keys"].size + inp["ivs"].size)
        else:
            call = lambda: backend_cuda.encrypt_shared_iv(hi, iv, rk, out=ho)  # noqa: E731
            api = "backend_cuda.encrypt_shared_iv -> gaes_encrypt_shared_iv (pinned host buffers)"
            h2d = int(n * 16)
        for _ in range(2):
            call()
        if launched:
            dist.barrier()
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(ts) / len(ts), reduce_dev)
        ok &= bool(np.array_equal(ho[:4096], ch[:4096]))
        e2e = {"value": job_blocks * BYTES_PER_BLOCK / e2e_s / 1e9, "unit": "GB/s",
               "step_ms": [round(t * 1e3, 3) for t in ts], "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(n * 16), "api": api}
        del h_in, h_out

    # ---- drop-in contract: the 7-argument backend call the reference's
    # encrypt_batch makes (aes_cbc.py:352-355): pageable numpy buffers,
    # IVSet.rows-tiled IVs, tables as _encrypt_tables builds them.
    dropin = None
    if not args.no_e2e and cfg != 5 and rank == 0:
        n_d = min(n, 1 << 22)
        hp = p[:n_d].cpu().numpy()
        ivrows = np.tile(np.frombuffer(iv, np.uint8), (n_d, 1))
        tables = (rk,) + backend_cuda.standard_tables(False)  # what _encrypt_tables(key) hands over
        hout = np.empty_like(hp)
        backend_cuda.cbc_encrypt(hp, ivrows, *tables, hout)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            backend_cuda.cbc_encrypt(hp, ivrows, *tables, hout)
            ts.append(time.perf_counter() - t0)
        ok &= bool(np.array_equal(hout[:4096], ch[:4096]))
        dropin = {"value": round(n_d * BYTES_PER_BLOCK / statistics.median(ts) / 1e9, 2), "unit": "GB/s",
                  "blocks": n_d, "h2d_bytes_per_step": int(n_d * 16), "d2h_bytes_per_step": int(n_d * 16),
                  "api": "backend_cuda.cbc_encrypt(data, ivs, round_keys, sbox, mix_lut, shift_src, out), "
                         "pageable numpy buffers (reference backend contract)"}
    return e2e, dropin, ok


def roofline_for(args, n, ms_local, clocks, dev, local, step, launches):
    """Roofline of the dominant kernel: shared-memory lookups/s against the
    peak measured in this run (gaes_probe_lds_peak), with the nominal figure,
    the formulation probe, the DRAM traffic from profiles/traffic.json and
    the HBM fraction nested."""
    import ctypes

    import torch

    from paper_1506_08503_b200 import _lib
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    peaks = {}
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    per_gpu_blocks_s = n / (ms_local / 1e3)
    # which lookups the L1/shared data pipe serves: round 10's 16 S-box
    # fetches go through the texture path when the library says so
    tex_sbox = _lib.lib().gaes_uses_sbox_texture(local) == 1
    lds_per_block = T_LOOKUPS_PER_BLOCK if tex_sbox else LOOKUPS_PER_BLOCK
    lds_achieved = per_gpu_blocks_s * lds_per_block / 1e9
    lds_peak = sms * 32 * sm_mhz * 1e6 / 1e9
    hbm_achieved = per_gpu_blocks_s * HBM_BYTES_PER_BLOCK / 1e9
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(f"cfg{args.config}")
        except (OSError, ValueError):
            traffic = None
    probe = lds_measured = None
    # the host-side legs above leave the GPU idle; bring the clocks back to
    # the timed region's before measuring the roofline denominators
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 0.3:
        step()
        torch.cuda.synchronize()
    try:
        rate, pms = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().gaes_probe_round_rate(local, 256, ctypes.addressof(rate), ctypes.addressof(pms)))
        probe = rate.value / 1e9
        # the roofline denominator, measured on this GPU in this run: a
        # conflict-free LDS.32 stream on every lane of every SM
        _lib.check(_lib.lib().gaes_probe_lds_peak(local, 4096, ctypes.addressof(rate), ctypes.addressof(pms)))
        lds_measured = rate.value / 1e9
    except Exception:  # pragma: no cover - informational only
        pass
    peak = lds_measured or lds_peak
    per_step = max(1, launches // max(1, args.steps))
    step()
    torch.cuda.synchronize()
    kernel = _lib.last_kernel()  # the step's kernel: k_blocks (large batches), k_blocks_small, k_many_key
    return {
        "bound": "smem", "kernel": kernel,
        "achieved": round(lds_achieved, 2), "peak": round(peak, 2), "unit": "Glookup/s",
        "frac": round(lds_achieved / peak, 4), "traffic": traffic,
        "traffic_unit": "GB per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, profiles/traffic.json)",
        # a step may be several launches (device-API calls are cut into
        # 2^28-block texture segments: config 5 = 4 launches per step)
        "algorithmic_gb_per_launch": round(n * HBM_BYTES_PER_BLOCK / per_step / 1e9, 4),
        "launches_per_step": per_step,
        "per_block": (f"{lds_per_block} conflict-free 4-B LDS table lookups per 16-B block (rounds 1-9)"
                      + (" + 16 S-box byte fetches on the TEX pipe (round 10)" if tex_sbox else
                         " incl. round 10's 16 S-box lookups")),
        "lookups_per_block": {"shared_memory": lds_per_block, "texture": LOOKUPS_PER_BLOCK - lds_per_block},
        "binding_note": ("the L1 data path is shared by the shared-memory T-table lookups (LSU side) and the "
                         "S-box / input texture fetches (TEX side); ncu: LSU wavefronts 96 %, TEX wavefronts 84 %, "
                         "l1tex__throughput 98 % (profiles/r1_final_ttable_ncu_summary.md); the per-instruction "
                         "attribution of the shared-load 'bank conflicts' ncu reports is in "
                         "profiles/r2/bank_conflicts.md" if tex_sbox else "ncu: L1 LSU data pipe 96 % busy"),
        "peak_source": ("measured: gaes_probe_lds_peak (k_lds_peak, conflict-free LDS.32 stream on every lane, "
                        f"{sms} SMs x 1024 threads) in this run; MEASURED_PEAKS.json has no shared-memory figure"
                        if lds_measured else "nominal (probe unavailable): 32 LDS lanes/clk/SM x SMs x SM clock"),
        "nominal_peak": round(lds_peak, 2),
        "nominal_frac": round(lds_achieved / lds_peak, 4),
        "nominal_note": f"{sms} SMs x 32 lanes/clk x {sm_mhz:.0f} MHz (median SM clock sampled during the timed region)",
        "probe_round_rate": round(probe * lds_per_block / LOOKUPS_PER_BLOCK, 2) if probe else None,
        "probe_frac": round(lds_achieved / (probe * lds_per_block / LOOKUPS_PER_BLOCK), 4) if probe else None,
        "probe_note": "k_round_probe: same round function (same S-box path) on register-resident states, no HBM "
                      "(formulation ceiling, in shared-memory lookups/s)",
        "hbm": {"achieved": round(hbm_achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(hbm_achieved / hbm_peak, 4),
                "per_block": f"{HBM_BYTES_PER_BLOCK} B (16 read + 16 written)",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
    }


def shard_digests(cfg: int, out, lo: int, hi: int, weak: bool, rank: int = 0) -> list:
    """SHA-256 of this rank's ciphertext: per piece (strong configs; the same
    8 pieces whatever N is, so N = 1 and N > 1 runs must print the same
    digests) or of the whole output (weak configs: every rank encrypts the
    workload, so every digest is the golden one for configs 1/2)."""
    spans = [(lo, hi)] if weak else [(a, b) for a, b in pieces(cfg) if lo <= a and b <= hi]
    if not spans:  # a rank count that cuts pieces: digest the rank's own range
        spans = [(lo, hi)]
    res = []
    with ThreadPoolExecutor(max_workers=2) as pool:
        futs = []
        for a, b in spans:
            host = out[a - lo:b - lo].cpu().numpy()  # the D2H of piece i overlaps the hash of piece i-1
            futs.append(((a, b), pool.submit(lambda h: hashlib.sha256(memoryview(h).cast("B")).hexdigest(), host)))
            if len(futs) > 2:
                futs[-3][1].result()
        for (a, b), f in futs:
            res.append({"blocks": [a, b], "rank": rank, "sha256": f.result()})
    return res


def _relaunch_under_torchrun(n: int) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this same
    command as N ranks, one per GPU, over 127.0.0.1 (what the driver does)."""
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
        return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main(argv=None):
    args = parse(argv)
    if args.gpus > 1 and "RANK" not in os.environ:
        return _relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        return run_reference_impl(args)

    import torch
    import torch.distributed as dist

    from paper_1506_08503_b200 import _lib, device
    from paper_1506_08503_b200.shard import bind_to_gpu_numa_node, gather_objects, max_over_ranks

    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    ndev = torch.cuda.device_count()
    if ndev == 0:
        print("bench.py: no CUDA device visible", file=sys.stderr)
        return 2
    # one rank per GPU (the driver's layout).  More ranks than GPUs happens
    # only in the 1-GPU test of the N > 1 path: ranks then share GPUs
    # round-robin (their kernels never wait on each other) and the timing
    # reductions go over gloo, since NCCL refuses two ranks on one GPU.
    gpu = local % ndev
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # torchrun, any world size
    backend = None
    if launched:
        backend = "nccl" if world <= ndev else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    reduce_dev = dev if backend == "nccl" else None
    # host side of this rank (pinned staging, copy threads) on the GPU's NUMA node
    numa_cpus = bind_to_gpu_numa_node(gpu) if world > 1 else None
    if args.variant:
        _lib.check(_lib.lib().gaes_set_variant(args.variant))
    # one process per GPU: host-buffer calls stay on this rank's device
    _lib.set_num_gpus(1)

    cfg = args.config
    w = WORKLOADS[cfg]
    weak = w["scaling"] == "weak"
    inp = make_inputs(cfg, rank, world, dev)
    p = inp["p"]
    n = p.shape[0]
    key, iv = inp["key"], inp["iv"]
    rk = device.expand_key(key, dev)  # GPU key schedule
    out = torch.empty_like(p)
    stream = torch.cuda.current_stream()

    if cfg == 5:
        d_keys = torch.from_numpy(inp["keys"]).to(dev)
        d_ivs = torch.from_numpy(inp["ivs"]).to(dev)
        rk_enc, rk_dec = device.expand_keys(d_keys)

        def step():
            device.many_key_encrypt(p, rk_enc, d_ivs, out=out)
    else:
        cipher = device.BlockCipher(rk, iv)

        def step():
            cipher.encrypt(p, out=out)

    small = n * 32 < 256 << 20  # working set below 2x L2
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if small else None

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    def capture(fn, k):
        """fn(i) for i < k as one CUDA graph (k launches); returns (graph, launches)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn(0)  # first-use work (smem opt-in, textures) stays outside the capture
        torch.cuda.current_stream().wait_stream(side)
        l0 = _lib.launch_count()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(k):
                fn(i)
        return g, _lib.launch_count() - l0

    graph = None
    if small:
        # Small batches (config 1): the K timed steps encrypt K distinct
        # copies of the batch -- a ring of inputs and outputs that one L2
        # flush before the region makes cold, so every step reads its input
        # from HBM ("inputs larger than L2") -- submitted as one CUDA graph of
        # K launches: the B200 way to issue a stream of small batches without
        # the host's per-launch enqueue cost (~4 us) on every step.
        ring_in = p.unsqueeze(0).repeat(args.steps, 1, 1)
        ring_out = torch.empty_like(ring_in)
        graph, graph_launches = capture(lambda i: cipher.encrypt(ring_in[i], out=ring_out[i]), args.steps)
        graph.replay()
        torch.cuda.synchronize()

    # ---- timed region: one pair of CUDA events on the launching stream around
    # K back-to-back steps (inputs larger than L2), or around the graph of K
    # steps on the cold ring (small batches)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(_smi_index(gpu)) as clk:
        # clocks are sampled every 100 ms; a timed region of K short steps can
        # be shorter than that, so the same kernel keeps running (untimed)
        # around it until the sampled window covers >= 0.5 s of load.
        clk.wait_first()
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.3:
            step()
            torch.cuda.synchronize()
        if launched:
            dist.barrier()
        torch.cuda.synchronize()
        mark = clk.mark()
        t_timed = time.perf_counter()
        if graph is not None:
            flush.fill_(1)  # evicts the whole ring (and keeps the GPU busy while the host enqueues)
            starts[0].record(stream)
            graph.replay()
            ends[0].record(stream)
            torch.cuda.synchronize()
            launches = graph_launches
        else:
            # one untimed step keeps the GPU busy while the host enqueues the
            # first timed step, so the start event does not absorb the Python
            # launch latency of an empty queue; the events bracket exactly K
            # steps, no event between launches (a launch starts its CTAs
            # while the previous one drains)
            step()
            launches0 = _lib.launch_count()
            starts[0].record(stream)
            for i in range(args.steps):
                step()
            ends[0].record(stream)
            torch.cuda.synchronize()
            launches = _lib.launch_count() - launches0
        ms = [starts[0].elapsed_time(ends[0]) / args.steps] * args.steps
        # ---- wall span: host barrier -> the last rank's
        # completion of K more steps, on the host's monotonic clock (shared
        # by the ranks of one node); events do not see skew between ranks.
        if launched:
            dist.barrier()
        t_b = time.perf_counter()
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step()
        torch.cuda.synchronize()
        t_e = time.perf_counter()
        span_s = max_over_ranks(t_e, reduce_dev) + max_over_ranks(-t_b, reduce_dev)
        # small batches, the other way round: each step its own stream launch
        # after an L2 flush, bracketed by its own events (reported beside the
        # value: includes the 4-6 us of stream-launch + event overhead that an
        # empty kernel shows the same way, profiles/r2/small_batches.md)
        stream_steps = None
        if small:
            s_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)]
            for i in range(args.steps):
                flush.fill_(i & 0xFF)
                s_ev[i][0].record(stream)
                step()
                s_ev[i][1].record(stream)
            torch.cuda.synchronize()
            sms_ = [a.elapsed_time(b) for a, b in s_ev]
            stream_steps = {"ms_per_step": round(sum(sms_) / len(sms_), 5),
                            "value": round(n * BYTES_PER_BLOCK / (sum(sms_) / len(sms_) / 1e3) / 1e9, 2),
                            "unit": "GB/s per GPU",
                            "note": "per step: L2 flush, event, one stream launch, event"}
        while time.perf_counter() - t_timed < 0.5:
            step()
            torch.cuda.synchronize()
        time.sleep(0.15)
    clocks = clk.summary(mark)
    clocks["window"] = "timed region + same-kernel soak to >= 0.5 s"
    clocks["throttled"] = any(r in clocks["reasons"] for r in
                              ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"))
    if graph is not None:
        assert torch.equal(ring_out[-1], ring_out[0])
        out = ring_out[0]
    ms_local = sum(ms) / len(ms)
    ms_step = max_over_ranks(ms_local, reduce_dev)
    job_blocks = n * world if weak else total_blocks(cfg, world)
    value = job_blocks * BYTES_PER_BLOCK / (ms_step / 1e3) / 1e9
    wall_span = {"ms_per_step": round(span_s * 1e3 / args.steps, 6),
                 "value": round(job_blocks * BYTES_PER_BLOCK * args.steps / span_s / 1e9, 2), "unit": "GB/s",
                 "note": ("host barrier -> last rank's completion of K steps (host monotonic clock, all ranks); "
                          + ("one graph replay of the K-step ring" if graph is not None else "back-to-back steps"))}

    # ---- verification (outside the timed region).  The GPU arm does not
    # touch the oracle: configs 1/2 use the reference recipe, so the whole
    # ciphertext must hash to the digest the reference's own compiled kernel
    # produced (tests/golden/golden.json); configs 3/4 are cross-checked
    # against the independent bitsliced formulation, config 5 against the
    # single-key kernel; every config must round-trip through decrypt.
    ch = out[:4096].cpu().numpy()
    check = {}
    digests = [] if args.no_digests and not weak else shard_digests(cfg, out, inp["lo"], inp["hi"], weak, rank)
    if cfg in (1, 2):
        with open(os.path.join(REPO, "tests", "golden", "golden.json")) as f:
            want = json.load(f)["digests"][str(n)]
        check["golden_match"] = digests[0]["sha256"] == want["sha256_c"] and key.hex() == want["key"]
        verified = bool(check["golden_match"])
        back = device.decrypt_blocks(out, rk, iv)
    elif cfg in (3, 4):
        m = min(n, 1 << 20)
        _lib.check(_lib.lib().gaes_set_variant(2))
        try:
            alt = device.encrypt_blocks(p[:m], rk, iv)
        finally:
            _lib.check(_lib.lib().gaes_set_variant(args.variant))
        check["bitsliced_cross_check_blocks"] = m
        verified = bool(torch.equal(alt, out[:m]))
        back = device.decrypt_blocks(out, rk, iv)
    else:
        bpk = inp["bpk"]
        verified = True
        for i in (0, inp["keys"].shape[0] - 1):
            rows = slice(i * bpk, (i + 1) * bpk)
            single = device.encrypt_blocks(p[rows], rk_enc[i].cpu().numpy(), inp["ivs"][i])
            verified &= bool(torch.equal(single, out[rows]))
        check["single_key_cross_check_keys"] = 2
        back = device.many_key_decrypt(out, rk_dec, d_ivs)
    verified &= bool(torch.equal(back, p))
    check["round_trip"] = bool(torch.equal(back, p))
    if cfg in (3, 4, 5):
        # an independent implementation on a seeded sample of this rank's
        # blocks: OpenSSL's AES-128-ECB of P ^ IV (pinned to the reference's
        # config-1 digest in tests/test_gpu_fullsize.py); not the oracle
        ossl = openssl_sample_check(inp, p, out, cfg)
        if ossl is not None:
            check["openssl_sample_blocks"] = ossl[1]
            verified &= ossl[0]

    # decrypt throughput (reported, not the metric): same discipline
    def dstep():
        if cfg == 5:
            device.many_key_decrypt(out, rk_dec, d_ivs, out=back)
        else:
            cipher.decrypt(out, out=back)
    for _ in range(3):
        dstep()
    torch.cuda.synchronize()
    dreps = max(3, min(args.steps, 10))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if small:
        ring_back = torch.empty_like(ring_out)
        dgraph, _ = capture(lambda i: cipher.decrypt(ring_out[i], out=ring_back[i]), args.steps)
        dgraph.replay()
        flush.fill_(7)
        ev0.record(stream)
        dgraph.replay()
        ev1.record(stream)
        torch.cuda.synchronize()
        dec_ms = ev0.elapsed_time(ev1) / args.steps
        assert torch.equal(ring_back[-1], p)
        del ring_back
    else:
        dstep()
        ev0.record(stream)
        for _ in range(dreps):
            dstep()
        ev1.record(stream)
        torch.cuda.synchronize()
        dec_ms = ev0.elapsed_time(ev1) / dreps
    dec_gbs = n * BYTES_PER_BLOCK / (dec_ms / 1e3) / 1e9
    del back

    # ---- e2e legs through the public host-buffer API
    e2e, dropin, ok = host_api_legs(args, inp, p, n, iv, rk, ch, world, rank, reduce_dev, launched)
    verified &= ok

    # ---- roofline of the dominant kernel (k_blocks encrypt)
    roofline = roofline_for(args, n, ms_local, clocks, dev, gpu, step, launches)

    cpu = None
    openssl = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_seconds)
        openssl = openssl_rate(key, iv)
        try:
            cpu["reference_api_e2e_cfg1"] = reference_api_e2e(key, iv)
        except Exception as e:  # pragma: no cover - informational only
            cpu["reference_api_e2e_cfg1"] = {"unavailable": f"{type(e).__name__}: {e}"}

    all_digests = gather_objects({"rank": rank, "verified": verified, "digests": digests})
    if rank == 0:
        verified_all = all(d["verified"] for d in all_digests)
        if weak and cfg in (1, 2):
            verified_all &= all(x["sha256"] == digests[0]["sha256"] for d in all_digests for x in d["digests"])
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None, "dtype": "u8",
            "data": ("synthetic: the reference bench recipe (numpy default_rng(2016): key, iv, uniform bytes), "
                     "copied to HBM before timing" if cfg in (1, 2)
                     else "synthetic (seeded, generated on device in 2^22-block chunks)"),
            "config": config_dict(cfg, world),
            "dist": {"backend": backend, "ranks": world, "gpus_visible": ndev,
                     "host_cpus": (f"{len(numa_cpus)} CPUs local to the GPU" if numa_cpus else "all")},
            "gpu_launches": launches, "wall_span": wall_span, "stream_launch_steps": stream_steps,
            "roofline": roofline, "e2e": e2e,
            "e2e_dropin": dropin, "cpu_baseline": cpu, "cpu_openssl": openssl, "clocks": clocks,
            "decrypt_gbs_per_gpu": round(dec_gbs, 2), "verified": bool(verified_all), "verification": check,
            "digests": sorted((x for d in all_digests for x in d["digests"]), key=lambda x: (x["blocks"], x["rank"])),
            "step_ms": [round(x, 4) for x in ms],
        }
        print(json.dumps(line))
        verified = verified_all
    if launched:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if verified else 1


if __name__ == "__main__":
    sys.exit(main())
