#!/usr/bin/env python
"""Benchmark: MCTS leaf pipeline (rebuild -> all-rule e-match -> OCF extraction) on B200.

BASELINE.json metric: "MCTS leaf extractions/sec + e-match matches/sec at 1/2/4/8 B200 vs
CPU ref". Headline workload: configs[2], the ResNeXt-50 analog with the multi-pattern rules and
batched leaf extraction -- the config the 1/2/4/8-GPU figure is quoted on. A *step* is one MCTS
simulation step over a batch of leaves: every leaf's dirty e-graph (left by apply_rule's unions)
is rebuilt, matched against all 22 TASO-analog rules (20 single + 2 multi-pattern joins) and
OCF-extracted; under torchrun the per-leaf results are all-gathered over NCCL (the MCTS exchange
of rewards / best costs). The other four BASELINE leaf sets are measured the same way into
``per_config``; ``mcts`` times the search itself (configs[1], NasRNN) on the device and on the
CPU reference engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--model M] [--impl ours|reference]

The leaves are the reference's own rollout states (tests/golden/bench_<model>.npz, made by
tests/golden/make_bench_leaves.py), replicated to B leaves per rank with a per-rank rotation.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MCTS leaf extractions/sec + e-match matches/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "leaf extractions/s"


def load_golden_leaves(model: str):
    """Fallback leaf set: the analog's reference rollout states from tests/golden/analog_<model>."""
    import gzip

    from paper_2410_05534_b200.arena import LeafState
    from paper_2410_05534_b200.symtab import NO_MATCH_CODE

    g = json.load(gzip.open(ROOT / "tests" / "golden" / f"analog_{model}.json.gz"))
    st = g["symtab"]
    leaves = [LeafState.from_json(c["state"]) for c in g["cases"]]
    symarr = {k: np.array(st[k], np.int32 if k == "params" else np.uint32)
              for k in ("name", "arity", "rank", "poff", "params")}
    names = {n: i for i, n in enumerate(st["names"])}
    codes = {(type(v), v): i for i, v in enumerate(st["values"])}
    ref = np.array([float.fromhex(c["extract"]["ocf"]["cost"]) for c in g["cases"]])
    return (leaves, symarr, lambda n: names.get(n, -1), lambda v: codes.get((type(v), v), NO_MATCH_CODE), ref,
            {"model": model, "source": "golden", "symbols": st["symbols"], "values": st["values"]})


def load_leaves(model: str):
    from paper_2410_05534_b200.arena import LeafState

    path = ROOT / "tests" / "golden" / f"bench_{model}.npz"
    if not path.exists():
        return load_golden_leaves(model)
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    L = int(z["n_leaves"])
    nb, kb, ub = z["node_base"].astype(np.int64), z["kid_base"].astype(np.int64), z["id_base"].astype(np.int64)
    leaves = []
    for l in range(L):
        n0, n1, k0, k1, u0, u1 = nb[l], nb[l + 1], kb[l], kb[l + 1], ub[l], ub[l + 1]
        leaves.append(LeafState(z["hc_sym"][n0:n1], z["hc_koff"][n0 + l:n1 + l + 1], z["hc_kids"][k0:k1],
                                z["hc_cid"][n0:n1], z["hc_cost"][n0:n1], z["uf_parent"][u0:u1],
                                z["uf_rank"][u0:u1], int(z["root"][l])))
    symarr = {"name": z["sym_name"], "arity": z["sym_arity"], "rank": z["sym_rank"], "poff": z["sym_poff"],
              "params": z["sym_params"]}
    names = {n: i for i, n in enumerate(meta["names"])}
    codes = {(type(v), v): i for i, v in enumerate(meta["values"])}
    name_id = lambda n: names.get(n, -1)  # noqa: E731
    from paper_2410_05534_b200.symtab import NO_MATCH_CODE

    code = lambda v: codes.get((type(v), v), NO_MATCH_CODE)  # noqa: E731
    return leaves, symarr, name_id, code, z["ref_ocf"], meta


def measure_apply(ctx, leaves, B: int, rotate: int, symarr, name_id, code, meta, reps: int = 10):
    """k_apply (device apply loop) on the same leaves: every leaf applies one of its
    live rules (1..600 matches, the rollouts' own draw rule, seeded), timed alone with CUDA events
    (the apply reads the rebuilt state and rewrites the batch input, so repeats are identical)."""
    import torch

    from paper_2410_05534_b200.apply import LANG_TENSOR, COST_ANALYTIC, symbol_arrays
    from paper_2410_05534_b200.arena import Batch
    from paper_2410_05534_b200.pipeline import LeafPipeline

    if not meta.get("symbols"):
        return None
    n = len(leaves)
    packed = Batch([leaves[(rotate + i) % n] for i in range(B)]).pack_with_headroom(nodes=2048)
    pipe = LeafPipeline(ctx, symarr, rules(), name_id, code)
    b = pipe.load(packed)
    b.set_counts(packed["n_cnt"], packed["u_cnt"])
    pipe.rebuild()
    pipe.ematch()
    counts = pipe.match_counts()
    rng = np.random.default_rng(0)
    leaf_rule = np.full(B, 0xFFFFFFFF, np.uint32)
    for l in range(B):
        live = np.nonzero((counts[:, l] > 0) & (counts[:, l] <= meta.get("max_matches", 600)))[0]
        if live.size:
            leaf_rule[l] = int(rng.choice(live))
    poff, flat = symarr["poff"], symarr["params"]
    codes = [flat[poff[i]:poff[i + 1]] for i in range(len(symarr["name"]))]
    sa = symbol_arrays(symarr["name"], symarr["arity"], [s[2] for s in meta["symbols"]], codes, meta["values"])
    off, words = pipe.apply_programs(name_id, code)
    ctx.apply_setup(LANG_TENSOR, COST_ANALYTIC, 1e-9, sa, off, words)
    b.apply(leaf_rule)
    res = b.download_apply()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.apply(leaf_rule)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    st = b.download_state()
    reb = b.download_rebuild()
    ok = res["status"] == 0
    out = {"kernel_ms": ms, "leaf_applies_per_s": B / (ms / 1e3), "leaves": B,
           "rule_choice": "uniform over each leaf's rules with 1..600 matches (seed 0)",
           "status_counts": {str(k): int(v) for k, v in zip(*np.unique(res["status"], return_counts=True))},
           "matches_applied": int(res["report"][ok, 0].sum()),
           "changed_leaves": int(res["report"][ok, 1].sum()),
           "cycles_filtered": int(res["report"][ok, 2].sum()), "shape_filtered": int(res["report"][ok, 3].sum()),
           "nodes_added": int((st["n"].astype(np.int64) - reb["n"].astype(np.int64))[ok].sum()),
           "parity": "tests/test_gpu_apply.py (reference rollouts, bit-exact)"}
    b.close()
    return out


def measure_fingerprint(ctx, batch, meta, reps: int = 10):
    """k_fingerprint (EGraph.fingerprint: the MCTS extraction-cache key) on the
    rebuilt leaves of the main batch, timed alone with CUDA events."""
    import torch

    from paper_2410_05534_b200.fingerprint import key_tables

    if not meta.get("symbols"):
        return None
    ctx.fingerprint_setup(*key_tables([tuple(s) for s in meta["symbols"]]))
    batch.fingerprint()
    fp, status = batch.download_fingerprint()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        batch.fingerprint()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"kernel_ms": ms, "leaf_fingerprints_per_s": batch.n_leaves / (ms / 1e3),
            "distinct_fingerprints": int(len(np.unique(fp))), "status_nonzero": int(np.sum(status != 0)),
            "parity": "tests/test_gpu_fingerprint.py (reference fingerprints of 1,819 states, bit-exact)"}


def make_batch(leaves, B: int, rotate: int):
    from paper_2410_05534_b200.arena import Batch

    n = len(leaves)
    return Batch([leaves[(rotate + i) % n] for i in range(B)]).pack(), [(rotate + i) % n for i in range(B)]


def rules():
    from paper_2410_05534_b200.patterns import load_rules

    return load_rules("taso_analog")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def start(self):
        self._t.start()

    def stop(self):
        self._stop.set()
        self._t.join(timeout=6)

    def __enter__(self):
        self.start()
        return self

    def __exit__(self, *a):
        self.stop()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def algorithmic_bytes(view, packed, counts_by_rule, rules_c, join_src_words=0):
    """SURVEY.md 8(d) compulsory traffic: per leaf rebuild 44N+8C, extraction 20N+20C, e-match
    16N+8C+4*M*W (N live e-nodes, C classes, M matches, W words). SURVEY charges the e-match view
    per pattern; k_ematch matches every pattern of a leaf in one CTA from one staged copy of the
    view, so it is charged once per leaf here (the compulsory traffic of the fused kernel)."""
    L = packed["n_leaves"]
    nb = packed["node_base"].astype(np.int64)
    n_in = np.diff(nb)
    N = view["n"].astype(np.int64)
    C = view["C"].astype(np.int64)
    b_rebuild = int(np.sum(44 * n_in + 8 * C))
    b_extract = int(np.sum(20 * N + 20 * C))
    b_ematch = int(np.sum(16 * N + 8 * C))   # the fused k_ematch reads a leaf's view once for all patterns
    b_join = 0
    for r, cnt in zip(rules_c, counts_by_rule):
        W = len(r.pattern_ids) + len(r.var_names) + len(r.pvar_names)
        if r.multi:   # join: read the source match lists, write the joined records
            b_join += int(4 * W * int(cnt.sum()))
        else:
            b_ematch += int(4 * W * int(cnt.sum()))
    b_join += 4 * int(join_src_words)   # the joins read their sources' match lists
    return {"rebuild": b_rebuild, "ematch": b_ematch, "join": b_join, "extract": b_extract}


def cpu_baseline(leaves, symarr, rules_c, budget_s: float = 15.0, threads: int = 0):
    """The oracle port on host cores: bounded sample of the same per-leaf pipeline."""
    from oracle import oracle as O
    from paper_2410_05534_b200.arena import Batch

    threads = threads or len(os.sched_getaffinity(0))
    done, t_total, reps = 0, 0.0, 0
    sample = len(leaves)                      # every distinct reference leaf of the workload
    packed = Batch(leaves[:sample]).pack()
    while t_total < budget_s and reps < 1000:
        t0 = time.perf_counter()
        O.pipeline(packed, symarr, rules_c, "ocf", threads)
        t_total += time.perf_counter() - t0
        done += sample
        reps += 1
    return done / t_total, threads, f"{sample} distinct leaves x {reps} reps ({t_total:.1f}s of CPU pipeline)"


def full_cpu_baseline(model, leaves, symarr, rules_c, meta, ref_ocf, budget_s: float = 8.0) -> dict:
    """the C port of the reference at all host cores (``value``) and at one core,
    plus the reference's own Python (baseline/_ref or the source tree) at one core and at all cores
    (a multiprocessing pool sharding leaves) on a bounded sample of the same leaves; the host's
    CPU model. The reference Python is far slower than the port, so ratios against ``value`` are
    conservative."""
    from oracle.ref_pipeline import cpu_model, host_cores, time_reference

    cores = host_cores()
    v_all, _, sample = cpu_baseline(leaves, symarr, rules_c, budget_s=budget_s, threads=cores)
    v_one, _, sample1 = cpu_baseline(leaves, symarr, rules_c, budget_s=budget_s, threads=1)
    out = {"value": v_all, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
           "one_core": {"value": v_one, "cores": 1, "sample": sample1},
           "cpu_model": cpu_model(), "workload": f"{model} leaf pipeline (rebuild + 22-rule joint_match + OCF)"}
    try:
        from oracle.mcts_ref import import_reference

        import_reference()
        from paper_2410_05534_b200.cost_model import CostModelConfig
        from oracle.ref_pipeline import leaf_pipeline

        text = (ROOT / "paper_2410_05534_b200" / "rules" / "taso_analog.rules").read_text()
        E, R, X, T = import_reference()
        _, cost0 = leaf_pipeline(leaves[0], meta["symbols"], R.parse_rules(text), CostModelConfig())
        r1 = time_reference(leaves, meta["symbols"], text, CostModelConfig(), budget_s=budget_s, workers=1)
        rn = time_reference(leaves, meta["symbols"], text, CostModelConfig(), budget_s=budget_s, workers=cores)
        out["reference_python"] = {"one_core": r1["value"], "all_cores": rn["value"], "cores": cores,
                                   "sample": f"{r1['leaves']} / {rn['leaves']} leaves in {budget_s:.0f}s",
                                   "cost_check": float(cost0) == float(ref_ocf[0]),
                                   "note": "the reference's own Python (esat.egraph.rebuild, rewrite.joint_match, "
                                           "extraction.extract_ocf_greedy) on the same leaves"}
    except ImportError as exc:
        out["reference_python"] = {"unavailable": str(exc)}
    return out


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the oracle port) on the
    box's host cores, on the same workload/metric; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    leaves, symarr, name_id, code, ref_ocf, meta = load_leaves(args.model)
    from paper_2410_05534_b200.pipeline import compile_rules

    _, rules_c = compile_rules(rules(), name_id, code)
    from oracle import oracle as O
    from paper_2410_05534_b200.arena import Batch

    threads = len(os.sched_getaffinity(0))
    sample = len(leaves)                      # every distinct reference leaf per step
    packed = Batch(leaves[:sample]).pack()
    for _ in range(args.warmup):
        O.pipeline(packed, symarr, rules_c, "ocf", threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.pipeline(packed, symarr, rules_c, "ocf", threads)
    dt = time.perf_counter() - t0
    v = sample * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
            "data": "synthetic (reference-generated MCTS rollout leaves)",
            "config": {"workload": f"{args.model} analog, MCTS leaf step (rebuild + 22-rule e-match + OCF), "
                                   f"CPU oracle port, {sample} leaves/step", "model": args.model,
                       "global_batch": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} leaves per step x {args.steps} steps",
                             "note": "C port of the reference algorithm (oracle/esat_oracle.c, pinned to the "
                                     "reference's goldens); the reference's own Python is ~100x slower "
                                     "(bench.py cpu_baseline.reference_python), so ratios against this arm are "
                                     "conservative"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure_config(ctx, stream, dev, model, B, steps, warmup, world, rank, e2e_steps, ocf_pool, clocks=None):
    """One leaf set through the pipeline: warm-up + parity, timed steps (device events, max over
    ranks), every kernel timed alone, the e2e loop through the C-ABI with pinned host buffers."""
    import torch
    import torch.distributed as dist

    from paper_2410_05534_b200 import native
    from paper_2410_05534_b200.parallel import allgather_leaf_results
    from paper_2410_05534_b200.pipeline import LeafPipeline

    leaves, symarr, name_id, code, ref_ocf, meta = load_leaves(model)
    pipe = LeafPipeline(ctx, symarr, rules(), name_id, code, method="ocf", pool_entries_per_node=ocf_pool)
    packed, src_idx = make_batch(leaves, B, rotate=rank * B)  # contiguous shard of the global leaf sequence
    batch = pipe.load(packed)
    ctx.reset_extract_lanes()    # a new leaf set: k_extract's lane groups are re-tuned on it
    for _ in range(max(warmup, 3)):
        pipe.step()
    torch.cuda.synchronize()
    ext = batch.download_extract()   # tunes the lane-group width (native.Context.tune_extract_lanes)
    pipe.step()                      # the parity-checked step runs with the tuned width
    ext = batch.download_extract()
    while pipe.grow_pool(ext):   # size the OCF history pools once, outside timing
        pipe.step()
        ext = batch.download_extract()
    exp = np.asarray(ref_ocf)[src_idx]
    parity_ok = bool(np.all(ext["status"] == 0) and np.array_equal(ext["root_cost"].view(np.uint64),
                                                                      exp.view(np.uint64)))
    view = batch.download_rebuild()
    view.update(batch.download_view())
    counts = pipe.match_counts()
    total_matches = int(counts.sum())
    src_words = 0
    for r in pipe.joins:
        for pid, prog in zip(r.pattern_ids, r._programs):
            _, _, c_src = batch.download_matches(pid)
            src_words += int(c_src.sum()) * (1 + int(prog[1]) + int(prog[2]))
    abytes = algorithmic_bytes(view, packed, counts, pipe.rules, src_words)

    res_cost = torch.empty(B, dtype=torch.float64, device=dev)
    res_stat = torch.empty(B, dtype=torch.int32, device=dev)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    stage_ms = {"rebuild": 0.0, "ematch": 0.0, "join": 0.0, "extract": 0.0}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(steps):
        e = ev[k]
        e[0].record(stream)
        pipe.rebuild()
        e[1].record(stream)
        ctx.fork()                # side stream: OCF extraction overlaps e-match + join
        pipe.match()
        e[2].record(stream)
        pipe.join()
        e[3].record(stream)
        pipe.extract_async()
        ctx.wait_async()
        e[4].record(stream)
        if world > 1:  # MCTS exchange: every rank needs every leaf's reward/cost
            batch.copy_results(res_cost.data_ptr(), res_stat.data_ptr())
            allgather_leaf_results(res_cost, res_stat)
    t_end.record(stream)
    torch.cuda.synchronize()
    if clocks is not None:
        clocks.stop()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    for e in ev:
        stage_ms["rebuild"] += e[0].elapsed_time(e[1])
        stage_ms["ematch"] += e[1].elapsed_time(e[2])
        stage_ms["join"] += e[2].elapsed_time(e[3])
        stage_ms["extract"] += e[3].elapsed_time(e[4])

    # every kernel alone on its own launches (same inputs, outside the timed region): the roofline
    # and the dominant kernel use these; stage_ms above are the overlapped in-step intervals
    def time_alone(fn, reps):
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        x0.record(stream)
        for _ in range(reps):
            fn()
        x1.record(stream)
        torch.cuda.synchronize()
        return x0.elapsed_time(x1) / reps

    reps = max(3, min(20, steps // 5))
    kernel_ms = {"rebuild": time_alone(pipe.rebuild, reps), "ematch": time_alone(pipe.match, reps),
                 "join": time_alone(pipe.join, reps), "extract": time_alone(pipe.extract, reps)}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- e2e through the public API with host buffers (pinned), per step: H2D arena, 4 launches,
    #      D2H root costs + statuses ----
    pinned = {}
    for k, v in packed.items():
        pinned[k] = torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy() if isinstance(v, np.ndarray) else v
    h2d = sum(int(pinned[k].nbytes) for k in ("hc_sym", "hc_koff", "hc_kids", "hc_cid", "hc_cost", "uf_parent",
                                             "uf_rank", "root"))
    outs = [(torch.empty(B, dtype=torch.float64).pin_memory().numpy(),
             torch.empty(B, dtype=torch.int32).pin_memory().numpy()) for _ in range(2)]
    d2h = outs[0][0].nbytes + outs[0][1].nbytes
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # two device batches alternate so step i+1's H2D upload (copy engine) overlaps step i's
    # kernels; every step still uploads its own inputs and reads back its own results
    ctx2 = native.Context(ctx.device)   # its own stream: the two batches' steps overlap
    if ctx.extract_lanes:                # the same extraction lane width as the tuned context
        ctx2.set_extract_lanes(ctx.extract_lanes)
    pipe2 = LeafPipeline(ctx2, symarr, rules(), name_id, code, method="ocf", pool_entries_per_node=pipe.pool,
                         pool_bitsets_per_node=pipe.pool_bitsets)
    batch2 = pipe2.load(packed)
    pipe2.step()
    torch.cuda.synchronize()
    pipes = [(pipe, batch), (pipe2, batch2)]
    t0 = time.perf_counter()
    pending = None
    for i in range(e2e_steps):
        pp, bb = pipes[i % 2]
        bb.upload(pinned)
        pp.step()
        if pending is not None:
            pending[0].download_extract_small(*pending[1])
        pending = (bb, outs[i % 2])
    pending[0].download_extract_small(*pending[1])
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    batch2.close()
    ctx2.close()
    n_nodes = np.diff(packed["node_base"].astype(np.int64))
    peak, _ = peaks()
    return {"model": model, "value": B * world * steps / (ms / 1e3), "ms_per_step": ms / steps,
            "e2e": {"value": B * world * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "kernel_ms": kernel_ms, "stage_ms_in_step": {k: v / steps for k, v in stage_ms.items()},
            "matches_per_step": total_matches * world,
            "matches_per_s": total_matches * world * steps / (ms / 1e3),
            "ematch_matches_per_s": total_matches * world / ((kernel_ms["ematch"] + kernel_ms["join"]) / 1e3),
            "rebuilds_per_s": B * world / (kernel_ms["rebuild"] / 1e3),
            "extractions_per_s": B * world / (kernel_ms["extract"] / 1e3),
            "roofline_frac": {k: abytes[k] / (kernel_ms[k] / 1e3) / 1e9 / peak for k in abytes},
            "algorithmic_bytes": abytes,
            "parity_vs_reference": parity_ok,
            "extract_lanes": ctx.extract_lanes, "extract_level_width": ctx.extract_width,
            "parity_detail": {"status_nonzero": int(np.sum(ext["status"] != 0)),
                              "cost_mismatch": int(np.sum(ext["root_cost"].view(np.uint64) != exp.view(np.uint64))),
                              "ocf_pool_entries_per_node": pipe.pool, "ocf_pool_bitsets_per_node": pipe.pool_bitsets},
            "leaves_per_rank": B, "distinct_leaves": len(leaves), "nodes_per_leaf_mean": float(n_nodes.mean()),
            "arena_mb": packed["hc_sym"].nbytes * 7 / 1e6,
            "_keep": (leaves, symarr, name_id, code, ref_ocf, meta, pipe, batch)}


def measure_mcts(ctx, budget: int = 128, batch: int = 32, node_limit: int = 800) -> dict:
    """configs[1]: the search itself. One run_search (budget iterations, batch 32, depth 10) from the
    NasRNN analog's initial e-graph on the device engine, and the same search on the CPU reference
    engine (oracle/mcts_ref.py: the reference's own apply_rule / is_rule_applicable /
    extract_ocf_greedy, all host cores) -- iterations/s of both and whether their trees agree. The
    node limit is the MCTS golden case's (tests/golden/mcts/nasrnn_c2.json): at 2000 the reference
    needs tens of minutes for one multi-pattern explosion."""
    import random

    from paper_2410_05534_b200 import analogs
    from paper_2410_05534_b200 import tensor_ir as T
    from paper_2410_05534_b200.cost_model import CostModelConfig
    from paper_2410_05534_b200.mcts import DeviceEngine, MctsConfig, SearchNode, run_search
    from paper_2410_05534_b200.patterns import load_rules
    from paper_2410_05534_b200.symtab import SymbolTable

    cfg = MctsConfig(budget=budget, node_limit=node_limit, seed=0, batch=batch, max_sim_steps=10)
    cost = CostModelConfig()
    rules_ = load_rules("taso_analog")

    def search(engine, eg):
        rng = random.Random(cfg.seed)
        (state,), c0, n, _, app = engine.evaluate([engine.initial(eg)])
        root = SearchNode(state, float(c0[0]), int(n[0]))
        root.b = {r for r in range(len(rules_)) if not app[0, r]}
        t0 = time.perf_counter()
        best = run_search(root, engine, len(rules_), cfg, rng)
        dt = time.perf_counter() - t0
        stats = {r: (ch.v.hex() if isinstance(ch.v, float) else ch.v, ch.n, ch.s) for r, ch in root.children.items()}
        return dt, best, stats

    eg = T.graph_to_egraph(analogs.build_analog("nasrnn", T.GraphBuilder))
    dev_engine = DeviceEngine(rules_, SymbolTable(), eg.language, cost, ctx=ctx)
    search(dev_engine, T.graph_to_egraph(analogs.build_analog("nasrnn", T.GraphBuilder)))   # warm-up
    dt_dev, best_dev, stats_dev = search(dev_engine, eg)
    out = {"workload": f"nasrnn analog run_search: budget {budget}, batch {batch}, depth 10, node limit {node_limit}, "
                       f"seed 0",
           "device_iterations_per_s": budget / dt_dev, "device_s": dt_dev, "best_rule": best_dev,
           "apply_regrows": dev_engine.regrows, "apply_presized": dev_engine.presized}
    try:
        from oracle.mcts_ref import ReferenceEngine, import_reference
        from oracle.ref_pipeline import host_cores

        E, R, X, Tr = import_reference()
        text = (ROOT / "paper_2410_05534_b200" / "rules" / "taso_analog.rules").read_text()
        ref_engine = ReferenceEngine(text, cost, workers=host_cores())
        try:
            dt_ref, best_ref, stats_ref = search(ref_engine, Tr.graph_to_egraph(analogs.build_analog("nasrnn",
                                                                                                  Tr.GraphBuilder)))
        finally:
            ref_engine.close()
        out.update({"cpu_engine_iterations_per_s": budget / dt_ref, "cpu_engine_s": dt_ref,
                    "cpu_engine_cores": host_cores(), "speedup": dt_ref / dt_dev,
                    "tree_equal": stats_dev == stats_ref and best_dev == best_ref})
    except ImportError as exc:
        out["cpu_engine"] = {"unavailable": str(exc)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=16384,
                    help="leaves per rank per step (SURVEY §8(d) C3: batches of 256..16k leaves)")
    ap.add_argument("--config-batch", type=int, default=4096, help="leaves per rank per step of the per_config sweep")
    ap.add_argument("--model", default="resnext50",
                    choices=["nasrnn", "bert", "resnext50", "inception_v3", "nasnet_a"],
                    help="headline leaf set: configs[2] ResNeXt-50 by default; the other BASELINE analogs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per_config sweep of the other leaf sets")
    ap.add_argument("--no-mcts", action="store_true", help="skip the MCTS search measurement")
    ap.add_argument("--config-steps", type=int, default=20)
    ap.add_argument("--quick", action="store_true", help="A/B timing only: skip the fingerprint and apply keys")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--ocf-pool", type=float, default=32.0,
                    help="OCF history pool entries per e-node (grown automatically if too small)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2410_05534_b200 import native

    ctx = native.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    B, K = args.batch, args.steps
    clk = Clocks(local)
    head = measure_config(ctx, stream, dev, args.model, B, K, args.warmup, world, rank, args.e2e_steps, args.ocf_pool,
                          clocks=clk)
    leaves, symarr, name_id, code, ref_ocf, meta, pipe, batch = head.pop("_keep")
    fp_line = None if args.quick else measure_fingerprint(ctx, batch, meta)
    apply_line = None if args.quick else measure_apply(ctx, leaves, min(B, 4096), rank * B, symarr, name_id, code, meta)
    per_config = {}
    if not args.no_configs:
        for m in ("bert", "nasrnn", "resnext50", "inception_v3", "nasnet_a"):
            if m == args.model:
                continue
            r = measure_config(ctx, stream, dev, m, args.config_batch, args.config_steps, args.warmup, world, rank,
                               max(5, args.e2e_steps // 2), args.ocf_pool)
            r.pop("_keep")
            per_config[m] = r
    per_config[args.model] = {k: v for k, v in head.items()}
    for r in per_config.values():
        r.setdefault("leaves_per_rank", B)
    mcts = None
    if not args.no_mcts and rank == 0:
        mcts = measure_mcts(ctx)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    kernel_ms, abytes = head["kernel_ms"], head["algorithmic_bytes"]
    dom = max(kernel_ms, key=kernel_ms.get)
    achieved = abytes[dom] / (kernel_ms[dom] / 1e3) / 1e9
    traffic = None
    tr = ROOT / "profiles" / "traffic.json"
    trd = json.loads(tr.read_text()) if tr.exists() else {}
    traffic = trd.get(args.model, {}).get(dom) if isinstance(trd.get(args.model), dict) else None
    cpu = None
    if not args.no_cpu_baseline:
        from paper_2410_05534_b200.pipeline import compile_rules

        _, rules_c = compile_rules(rules(), name_id, code)
        cpu = full_cpu_baseline(args.model, leaves, symarr, rules_c, meta, ref_ocf)
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+u32", "data": "synthetic (reference-generated MCTS rollout leaves of the analog graph)",
        "config": {"workload": f"{args.model} analog (configs[2]: multi-pattern rules, batched leaf extraction) MCTS "
                               f"leaf step: rebuild + 22-rule e-match (20 single, 2 multi-pattern joins) + OCF "
                               f"extraction, {B} leaves/rank",
                   "model": args.model, "global_batch": B * world, "leaves_per_rank": B,
                   "distinct_leaves": head["distinct_leaves"], "nodes_per_leaf_mean": head["nodes_per_leaf_mean"],
                   "parallelism": f"leaf-sharded x{world} (NCCL all-gather of per-leaf results)",
                   "l2": f"inputs larger than L2 ({head['arena_mb']:.0f} MB leaf arena per rank)"},
        "matches_per_s": head["matches_per_s"], "matches_per_step": head["matches_per_step"],
        "rebuilds_per_s": head["rebuilds_per_s"], "extractions_per_s": head["extractions_per_s"],
        "ematch_matches_per_s": head["ematch_matches_per_s"],
        "kernel_ms": kernel_ms, "stage_ms_in_step": head["stage_ms_in_step"],
        "parity_vs_reference": head["parity_vs_reference"], "parity_detail": head["parity_detail"],
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_step": abytes[dom]},
        "roofline_by_kernel": {k: {"achieved_gbs": abytes[k] / (kernel_ms[k] / 1e3) / 1e9,
                                   "frac": abytes[k] / (kernel_ms[k] / 1e3) / 1e9 / peak,
                                   "traffic": trd.get(args.model, {}).get(k)
                                   if isinstance(trd.get(args.model), dict) else None}
                               for k in abytes},
        "extract_lanes": head["extract_lanes"], "extract_level_width": head["extract_level_width"],
        "per_config": {m: {k: r[k] for k in ("value", "ms_per_step", "e2e", "kernel_ms", "roofline_frac",
                                              "extract_lanes", "extract_level_width",
                                              "matches_per_s", "ematch_matches_per_s", "nodes_per_leaf_mean",
                                              "leaves_per_rank", "parity_vs_reference")}
                       for m, r in per_config.items()},
        "schedule": "k_rebuild -> [k_extract on a side stream || k_ematch -> k_join] -> join streams",
        "apply": apply_line,
        "fingerprint": fp_line,
        "mcts": mcts,
        "e2e": head["e2e"],
        "gpu_launches": pipe.LAUNCHES_PER_STEP * K,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
