#!/usr/bin/env python
"""Bench: sparse-FFN decode tokens/s on a BASELINE.json shape (default configs[1]:
ProSparse-Llama2-7B FFN stack, 32 layers d=4096 d_ff=11008, batch 1).

One step = one decode token through all L sparse-FFN layers (sequential
pipeline, ffn_exec.hpp:183-218), executed by ONE persistent cooperative launch
of the sm_100a executor (sg_ffn_forward_layers). Inputs/weights are resident in
HBM; the L layers touch ~2.3 GB per step (>> 126 MB L2), so every step streams
its bytes from HBM (no L2 flush needed; stated in `config`).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7b|mistral|13b|1layer]
  python bench.py --impl reference ...   # the reference CPU path (oracle/_ref)

N>1 (torchrun): the FFN intermediate dimension is sharded over ranks;
each layer ends with an NCCL all-reduce of the d-sized output.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)



# BASELINE.json configs (the shapes of paper_2603_14110_b200.model.CONFIGS, repeated here so
# the reference arm never imports this repo's package)
SHAPES = {
    "1layer": dict(d=4096, D=11008, L=1, act=0, model="single ReGLU FFN layer d=4096 d_ff=11008"),
    "7b": dict(d=4096, D=11008, L=32, act=0, model="ProSparse-Llama2-7B FFN stack"),
    "mistral": dict(d=4096, D=14336, L=32, act=1, model="TurboSparse-Mistral-7B FFN stack (dReLU)"),
    "13b": dict(d=5120, D=13824, L=40, act=0, model="ProSparse-Llama2-13B FFN stack"),
    "tiny": dict(d=512, D=1408, L=4, act=0, model="tiny test stack"),
}


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def touched_bytes(d, D, r, p, v):
    """algorithmic bytes of one layer for one token."""
    return 2 * r * d + 2 * D * r + 4 * D + 2 * d * p + 2 * d * v + 2 * d * v


def dense_bytes(d, D):
    return 3 * 2 * d * D


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0, period_ms=50):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        self.t.join(1)
        rows = [r for r in self.rows if len(r) >= 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    """Host CPU model and logical CPU count (SURVEY.md §8d asks for both)."""
    name = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    name = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    threads = os.environ.get("SPARSEGATE_THREADS", "unset")
    return f"{name} ({os.cpu_count()} logical CPUs, SPARSEGATE_THREADS={threads})"


# ---------------------------------------------------------------------------
# reference arm: the reference's own executor headers (oracle/_ref) on host cores
# ---------------------------------------------------------------------------
def _ref_layer_inputs(d, D, seed, rank, sparsity, calib_tokens=256, eval_tokens=16):
    """One layer of the bench workload built WITHOUT this repo's package (so nothing
    of ours is loaded in the reference arm), by the recipe of model.build_host_layer:
    weights from the reference's own make_synthetic_fixture (synthetic.hpp:80-108,
    via oracle/_ref), a rank-r truncated SVD of W_gate by a seeded randomized range
    finder (numpy; the reference's naive mode, factorization.hpp:93-144 with S = I),
    and the bias from the reference's own damage-weighted greedy calibration
    (calibration.hpp:61-205, via oracle/_ref) on the fixture's calibration tokens."""
    import oracle as O
    fx = O.ref_synthetic(d, D, calib_tokens, eval_tokens, 0.9, seed)
    G = fx["gate"].astype(np.float32)
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(G @ rng.standard_normal((d, rank + 8)).astype(np.float32))
    Q, _ = np.linalg.qr(G.T @ Q)
    Q, _ = np.linalg.qr(G @ Q)
    Ub, sv, Vt = np.linalg.svd(Q.T @ G, full_matrices=False)
    A = ((Q @ Ub[:, :rank]) * sv[None, :rank]).astype(np.float64)
    B = Vt[:rank].astype(np.float64)
    Xc = fx["calib"]
    scores = A @ (B @ Xc)
    gp, up = fx["gate"] @ Xc, fx["up"] @ Xc
    inner = np.maximum(gp, 0) * up
    weights = inner ** 2 * np.sum(fx["down"] ** 2, axis=0)[:, None]
    bias, _, _ = O.ref_greedy_calibrate(scores, weights, 8, sparsity)
    return fx["gate"], fx["up"], fx["down"], A, B, bias, np.ascontiguousarray(fx["eval"].T)


def run_reference(args, world, rank):
    """The reference's CPU executor (sparse_ffn_sequential, ffn_exec.hpp:183-218, f64 with
    its per-call validation) on the bench workload: every one of the L layers of the
    model is built (seeds 0..L-1, as our arm) and timed on its own eval tokens, tokens
    in parallel over all host threads (parallel_for, tools/sparsegate_main.cpp:241-259).
    A step is ntok tokens through all L layers; tokens/s = ntok / sum of layer times."""
    if rank != 0:
        return 0
    import concurrent.futures as cf

    import oracle as O

    cfg = SHAPES[args.config]
    d, D, L = cfg["d"], cfg["D"], cfg["L"]
    if args.layers:
        L = args.layers
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsgref.so not built"}))
        return 0
    cores = int(O.ref().sgref_thread_budget())
    ntok = max(1, min(cores, 16))
    k = max(1, min(args.steps, 3))
    w = 1
    t_build = time.time()
    per_layer = []
    chunk = max(1, min(8, (os.cpu_count() or 8) // 2))
    with cf.ThreadPoolExecutor(chunk) as ex:
        for l0 in range(0, L, chunk):
            # build a chunk of layers in parallel, then time them with the host idle
            built = list(ex.map(lambda l: _ref_layer_inputs(d, D, l, args.rank, args.sparsity),
                                range(l0, min(L, l0 + chunk))))
            for gate, up, down, A, B, bias, ev in built:
                ref = O.RefLayer(gate, up, down, A, B, bias, activation=cfg["act"])
                xs = np.ascontiguousarray(ev[:ntok])
                for _ in range(w):
                    ref.run(xs, pipeline=2)
                per_layer.append(sum(ref.run(xs, pipeline=2)[2] for _ in range(k)) / k)
                del ref
            del built
    step_s = float(sum(per_layer))
    tok_s = ntok / step_s
    line = {
        "impl": "reference", "metric": "sparse-FFN decode tokens/s", "value": tok_s,
        "unit": "tokens/s", "n_gpus": 0, "steps": k, "warmup": w,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1000.0 * step_s / ntok, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfg, args, L, 1),
        "per_layer_us": 1e6 * step_s / (ntok * L),
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{ntok} tokens (eval tokens of each layer, in parallel over "
                                   f"{cores} threads) through all {L} distinct layers, {k} timed "
                                   f"run(s) per layer after {w} warm-up; reference "
                                   f"sparse_ffn_sequential in f64 with its per-call validation; "
                                   f"inputs built in {time.time() - t_build:.0f} s, untimed"},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_config(cfg, args, L, world):
    """The `config` object of both arms (identical for the same command line)."""
    d, D = cfg["d"], cfg["D"]
    chain = getattr(args, "chain", 1)
    return {"workload": f"{cfg['model']}: {L} layers d={d} d_ff={D} r={args.rank} "
                        f"s={args.sparsity} natural sparsity 0.9, batch {max(1, args.batch)}, "
                        f"sequential pipeline, {'chained' if chain else 'unchained'} decode",
            "layers": L, "hidden": d, "inter": D, "rank": args.rank,
            "predicted_sparsity_target": args.sparsity, "batch": max(1, args.batch),
            "chain": {0: "unchained", 1: "raw y_l -> x_{l+1}", 2: "residual h_{l+1} + y_l"}[chain],
            "parallelism": f"d_ff-shard{world}" if world > 1 else "none"}


def cpu_baseline_for(cfg, host_layer0, args):
    """Rank-0 bounded sample of the reference CPU path on layer 0 (see run_reference)."""
    import oracle as O
    from paper_2603_14110_b200 import bf16_to_f64
    d, D, L = cfg["d"], cfg["D"], cfg["L"]
    if not O.ref_available():
        kind, cores = "port", 1
    else:
        kind, cores = "reference", int(O.ref().sgref_thread_budget())
    h = host_layer0
    gate, up = bf16_to_f64(h.gate), bf16_to_f64(h.up)
    down = np.ascontiguousarray(bf16_to_f64(h.down_t).T)
    A, B = bf16_to_f64(h.A), bf16_to_f64(h.B)
    bias = h.bias.astype(np.float32).astype(np.float64)
    ntok = max(1, min(cores, h.xs.shape[1]))
    xs = np.ascontiguousarray(h.xs[:, :ntok].T)
    if kind == "reference":
        ref = O.RefLayer(gate, up, down, A, B, bias, activation=cfg["act"])
        ref.run(xs[:1], 2)
        tot, reps = 0.0, 0
        while tot < 10.0 and reps < 8:
            _, _, el = ref.run(xs, 2)
            tot += el
            reps += 1
    else:
        t0 = time.perf_counter()
        reps = 1
        for t in range(ntok):
            O.sparse_ffn(gate, up, down, A, B, bias, xs[t])
        tot = time.perf_counter() - t0
    per = tot / (reps * ntok)
    return {"value": 1.0 / (per * L), "unit": "tokens/s", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"{reps} x {ntok} eval tokens through layer 0 of {L} (reference "
                      f"sparse_ffn_sequential, f64 incl. per-call validation, parallel_for over "
                      f"tokens); tokens/s = 1/(t_token_layer*{L})",
            "per_layer_us": per * 1e6}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_batch(args, cfg, host, layers, ctx, world, rank, local):
    """Batched decode (configs[4]): B tokens per step through the L layers, one
    sg_ffn_forward_batch per layer — for B >= 2 ONE persistent tcgen05 launch per layer
    (csrc/sg_batch_tc.cu) — the whole step captured in one CUDA graph. The dense
    comparator is the same kernel with every row (sg_ffn_forward_batch_dense)."""
    import ctypes as C

    import torch

    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import check
    lib = capi.lib()
    d, D, L, B = cfg["d"], cfg["D"], len(host), args.batch
    X = torch.tensor(np.stack([h.xs[:, :B].T for h in host]), dtype=torch.float32, device="cuda")
    Y = torch.zeros_like(X)
    stream = torch.cuda.Stream()

    chain = args.chain

    def layer_io(l):
        """(x, residual) device pointers of layer l under the bench's chain mode:
        0 independent batches, 1 x_{l+1} = y_l, 2 x_{l+1} = h_{l+1} + y_l."""
        if l == 0 or chain == 0:
            return X[l].data_ptr(), None
        if chain == 1:
            return Y[l - 1].data_ptr(), None
        return X[l].data_ptr(), Y[l - 1].data_ptr()

    def call(l, sh, dense=0):
        x, res = layer_io(l)
        # the next call's input (h_{l+1} + y_l or y_l) is known: this launch's y finishers
        # write its bf16 X^T too
        nxt, nxs = None, None
        if l + 1 < L and chain:
            nxt = layers[l + 1].handle
            nxs = C.c_void_p(X[l + 1].data_ptr()) if chain == 2 else None
        check(lib.sg_ffn_forward_batch_res(ctx.handle, layers[l].handle, C.c_void_p(x),
                                           C.c_void_p(res) if res else None, B,
                                           C.c_void_p(Y[l].data_ptr()), dense, nxt, nxs, C.c_void_p(sh)))

    arr = (C.c_void_p * L)(*[ly.handle.value for ly in layers])

    def step(sh, dense=0):
        if B == 1:
            # one token: the persistent single-token executor over the whole stack in one
            # launch (the headline path), dense comparator = its dense pipeline
            check(lib.sg_ffn_forward_layers(ctx.handle, arr, L, 0 if dense else 2,
                                            C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), chain,
                                            C.c_void_p(sh)))
            return
        for l in range(L):
            call(l, sh, dense)

    with torch.cuda.stream(stream):
        step(stream.cuda_stream)  # workspaces / attributes / tensor maps before capture
        step(stream.cuda_stream, 1)
    torch.cuda.synchronize()
    # union sizes per layer (roofline bytes), re-run un-captured
    pb = np.zeros(layers[0].local_inter, dtype=np.uint64)
    vb = np.zeros_like(pb)
    up, uv = [], []
    stats = (capi.sg_exec_stats * B)()
    for l in range(L):
        call(l, stream.cuda_stream)
        check(lib.sg_ctx_read_batch(ctx.handle, C.c_void_p(stream.cuda_stream), B, stats,
                                    pb.ctypes.data_as(C.c_void_p), vb.ctypes.data_as(C.c_void_p)))
        up.append(int((pb != 0).sum()))
        uv.append(int((vb != 0).sum()))

    def graph_of(dense):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(torch.cuda.current_stream().cuda_stream, dense)
        return g

    graph = graph_of(0)
    dgraph = graph_of(1)

    def timed(g, K, W, clocks=False):
        for _ in range(W):
            g.replay()
        torch.cuda.synchronize()
        sampler = ClockSampler(local) if clocks else None
        if sampler:
            time.sleep(0.15)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K, (sampler.stop() if sampler else None)

    ms, clocks = timed(graph, args.steps, args.warmup, clocks=True)
    ms_dense, _ = timed(dgraph, max(10, args.steps // 2), args.warmup)
    r = args.rank
    alg = sum(2 * r * d + 2 * D * r + 4 * D + 2 * d * p + 4 * d * v + 8 * d * B for p, v in zip(up, uv))
    dense_alg = L * (3 * 2 * d * D + 8 * d * B)
    hbm, hbm_kind = peaks()
    # e2e: pinned host tokens in, outputs back, through the same graph
    xh = torch.empty_like(X, device="cpu").pin_memory()
    xh.copy_(X)
    yh = torch.empty_like(Y, device="cpu").pin_memory()

    def e2e_step():
        X.copy_(xh, non_blocking=True)
        graph.replay()
        yh.copy_(Y, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for _ in range(3):
        e2e_step()
    ke = max(10, min(args.steps, 200))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(ke):
        e2e_step()
    t1.record()
    torch.cuda.synchronize()
    ms_e2e = t0.elapsed_time(t1) / ke
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_for(cfg, host[0], args)
        except Exception as e:  # report, never fake
            cpu = {"value": None, "error": str(e)[:200]}
    conf = bench_config(cfg, args, L, world)
    conf.update({"l2": "no flush: each step streams the union rows of %d distinct layers" % L,
                 "path": "B = 1: persistent single-token executor, one launch for the stack; "
                         "B >= 2: one tcgen05 launch per layer"})
    line = {
        "metric": "sparse-FFN decode tokens/s", "value": B * 1000.0 / ms, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": conf,
        "per_layer_us": ms * 1000.0 / L,
        "union_p_mean": float(np.mean(up)), "union_v_mean": float(np.mean(uv)),
        "roofline": {"bound": "hbm", "achieved": alg / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": alg / (ms * 1e-3) / 1e9 / hbm, "peak_kind": hbm_kind, "traffic": None,
                     "bytes_per_step": alg,
                     "kernel": "tc_kernel (csrc/sg_batch_tc.cu: tcgen05.mma + TMEM, TMA tiles)"
                               if B > 1 else "ffn_kernel<2> (persistent single-token executor)"},
        "dense": {"ms_per_step": ms_dense, "tokens_per_s": B * 1000.0 / ms_dense,
                  "per_layer_us": ms_dense * 1000.0 / L,
                  "achieved_gbs": dense_alg / (ms_dense * 1e-3) / 1e9,
                  "frac": dense_alg / (ms_dense * 1e-3) / 1e9 / hbm,
                  "sparse_speedup": ms_dense / ms,
                  "kernel": "tc_kernel dense mode (sg_ffn_forward_batch_dense)"},
        "e2e": {"value": B * 1000.0 / ms_e2e, "unit": "tokens/s", "h2d_bytes_per_step": L * B * d * 4,
                "d2h_bytes_per_step": L * B * d * 4, "ms_per_step": ms_e2e},
        "gpu_launches": args.steps * (1 if B == 1 else L),
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def near_threshold(host, ys_gpu, xs_in, sets, act, eps=2.0 ** -14):
    """Per-layer near-threshold diagnostics of the timed configuration:
    the f64 pre-activations of the bf16 weights on the token each layer saw, the size
    of the admissible band |pre| <= eps * sum|terms| (P) / |g| <= eps * sum|gate x| (V),
    and how many GPU decisions differ from the f64 sign (all must lie in the band)."""
    from paper_2603_14110_b200 import bf16_to_f64
    out = []
    for l, h in enumerate(host):
        x = np.asarray(xs_in[l], dtype=np.float64)
        A, B = bf16_to_f64(h.A), bf16_to_f64(h.B)
        bias = h.bias.astype(np.float32).astype(np.float64)
        t = B @ x
        pre = A @ t + bias
        sp = np.abs(A) @ np.abs(t) + np.abs(bias)
        G = bf16_to_f64(h.gate)
        g = G @ x
        sg = np.abs(G) @ np.abs(x)
        P_gpu, V_gpu = sets[l]
        P_ref = np.flatnonzero(pre > 0)
        band_p = np.abs(pre) <= eps * sp
        band_v = np.abs(g) <= eps * sg
        dP = np.setxor1d(P_ref, P_gpu)
        V_exp = P_gpu[g[P_gpu] > 0] if len(P_gpu) else P_gpu
        dV = np.setxor1d(V_exp, V_gpu)
        out.append(dict(band_p=int(band_p.sum()), band_v=int(band_v.sum()), flips_p=int(len(dP)),
                        flips_v=int(len(dV)), outside_band=int((~band_p[dP]).sum() + (~band_v[dV]).sum())))
    return {"eps": eps, "layers": len(out),
            "band_p_mean": float(np.mean([o["band_p"] for o in out])),
            "band_v_mean": float(np.mean([o["band_v"] for o in out])),
            "flips_p_total": int(sum(o["flips_p"] for o in out)),
            "flips_v_total": int(sum(o["flips_v"] for o in out)),
            "flips_outside_band": int(sum(o["outside_band"] for o in out))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="7b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--rank", type=int, default=256)
    ap.add_argument("--sparsity", type=float, default=0.5)
    ap.add_argument("--chain", type=int, default=2,
                    help="2 (default): layer l+1 reads h_{l+1} + y_l (the residual-stream decode "
                         "dependency: it cannot start before layer l's y exists); 1: reads y_l raw "
                         "(this synthetic FFN shrinks y ~100x per layer, so the operating point "
                         "drifts); 0: every layer reads its own token (the unchained line is "
                         "reported too)")
    ap.add_argument("--mode", default="stack", choices=["stack", "per-layer", "sharded"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-diag", action="store_true", help="skip the near-threshold diagnostics")
    ap.add_argument("--no-balance", action="store_true",
                    help="ascending neuron layout instead of the load-balanced order")
    ap.add_argument("--hot-rows", type=int, default=16,
                    help="gate rows per CTA fetched before the mask (sg_layer_set_hot_rows; 0 = off)")
    ap.add_argument("--no-graph", action="store_true",
                    help="per-layer mode: eager launches instead of one CUDA graph per step")
    ap.add_argument("--batch", type=int, default=0,
                    help="batched decode (configs[4]): B tokens per step through all layers")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import ctypes as C

    import torch

    # SG_BENCH_BACKEND / SG_BENCH_DEVICE: functional checks of the N>1 code path on a
    # one-GPU box (gloo, every rank on device 0); never used for timing claims
    local = int(os.environ.get("SG_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2603_14110_b200 import _capi as capi
    from paper_2603_14110_b200.ffn_exec import Context, Pipeline, check
    from paper_2603_14110_b200.model import build_host_model, upload

    t0 = time.time()
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(max(1, (os.cpu_count() or 8) // 8))
    except Exception:
        pass
    cfg, host = build_host_model(args.config, args.layers, rank=args.rank,
                                 sparsity=args.sparsity, workers=8,
                                 eval_tokens=max(16, args.batch))
    d, D, L = cfg["d"], cfg["D"], len(host)
    log(f"host model built in {time.time() - t0:.1f}s")
    # configs[0] is ONE layer (~70 MB touched < 126 MB L2): the step rotates over 4
    # device copies of it so every step streams its bytes from HBM
    copies = 4 if L == 1 else 1
    # batched decode (B >= 2): neurons by decreasing calibration activity (the batch's
    # survivor rows concentrate in the leading blocks; trailing blocks skip their down
    # rows); one token keeps the single-token executor's per-CTA balanced layout
    balance = False if args.no_balance else ("sorted" if args.batch > 1 else True)
    layers = [upload(h, d, D, cfg["act"], args.rank, device=local, shard_index=rank,
                     shard_count=world, balance=balance,
                     hot_rows=args.hot_rows) for h in host for _ in range(copies)]
    host_l = [h for h in host for _ in range(copies)]
    Ls = len(layers)  # layers per launch
    Dl = layers[0].local_inter
    ctx = Context(local, d, Dl, args.rank)
    lib = capi.lib()
    if args.batch > 0:
        return run_batch(args, cfg, host, layers, ctx, world, rank, local)
    arr = (C.c_void_p * Ls)(*[l.handle.value for l in layers])
    xs = torch.tensor(np.stack([h.x for h in host_l]), dtype=torch.float32, device="cuda")
    ys = torch.zeros_like(xs)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    # N > 1 (or --mode sharded): the C++ sharded step (csrc/sg_comm.cpp) — per-layer
    # launches on this rank's d_ff shard + one NCCL all-reduce per layer, from C++
    sharded = world > 1 or args.mode == "sharded"
    is_stack = args.mode == "stack" and not sharded
    if copies > 1:
        args.chain = 0  # rotated copies of one layer are independent
    chain = args.chain
    comm = None
    if sharded:
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib.sg_comm_unique_id(uid))
        if world > 1:
            obj = [bytes(uid)]
            torch.distributed.broadcast_object_list(obj, src=0)
            C.memmove(uid, obj[0], 128)
        comm = C.c_void_p()
        check(lib.sg_comm_create(local, world, rank, uid, C.byref(comm)))

    def step_stack(pipe=Pipeline.Sequential, ch=None, s=None):
        check(lib.sg_ffn_forward_layers(ctx.handle, arr, Ls, int(pipe), C.c_void_p(xs.data_ptr()),
                                        C.c_void_p(ys.data_ptr()), chain if ch is None else ch,
                                        C.c_void_p(sh if s is None else s)))

    def step_layers(pipe=Pipeline.Sequential, s=None):
        if sharded:
            check(lib.sg_ffn_forward_layers_sharded(ctx.handle, comm, arr, Ls, int(pipe),
                                                    C.c_void_p(xs.data_ptr()), C.c_void_p(ys.data_ptr()),
                                                    chain, C.c_void_p(sh if s is None else s)))
            return
        for l in range(Ls):
            src = ys[l - 1] if (chain == 1 and l > 0) else xs[l]
            check(lib.sg_ffn_forward_device(ctx.handle, layers[l].handle, int(pipe),
                                            C.c_void_p(src.data_ptr()),
                                            C.c_void_p(ys[l].data_ptr()), C.c_void_p(sh if s is None else s)))

    launches_per_step = 1 if is_stack else Ls

    def capture(fn):
        """fn(stream handle) replayed as one CUDA graph (warm call first: attributes,
        descriptor tables, NCCL communicator)."""
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs):
            fn(cs.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            fn(torch.cuda.current_stream().cuda_stream)
        return g

    graph_mode = "none"
    step = (lambda: step_stack()) if is_stack else (lambda: step_layers())
    graphs = {}
    if not args.no_graph and os.environ.get("SG_BENCH_BACKEND", "nccl") == "nccl":
        try:
            if is_stack:
                for ch in {chain, 0}:
                    graphs[ch] = capture(lambda s, ch=ch: step_stack(ch=ch, s=s))
                graph_mode = "stack launch captured in a CUDA graph"
            else:
                graphs[chain] = capture(lambda s: step_layers(s=s))
                graph_mode = "per-layer launches captured in one CUDA graph"
            step = graphs[chain].replay
        except Exception as e:  # report, keep eager
            log(f"graph capture failed, eager launches: {e}")

    def timed(fn, K, W, sample_clocks=False):
        for _ in range(W):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        sampler = ClockSampler(local) if sample_clocks else None
        if sampler:
            time.sleep(0.15)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(K):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        clocks = sampler.stop() if sampler else None
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, clocks

    ms, clocks = timed(step, args.steps, args.warmup, sample_clocks=True)
    unchained = None
    if is_stack and chain and 0 in graphs:
        ms_u, _ = timed(graphs[0].replay, max(10, args.steps // 2), args.warmup)
        unchained = {"ms_per_step": ms_u, "tokens_per_s": 1000.0 / ms_u,
                     "per_layer_us": ms_u * 1000.0 / Ls,
                     "note": "every layer reads its own token: layer l+1's x loads overlap "
                             "layer l's completion poll (not a real decode dependency)"}

    # per-layer stats (p, v) and index sets of the configuration just timed
    stats = (capi.sg_exec_stats * Ls)()
    sets = None
    if is_stack:
        if Ls <= 64 and not args.no_diag:
            check(lib.sg_ctx_enable_stack_sets(ctx.handle, 1))
        step_stack()
        check(lib.sg_ctx_read_stack_stats(ctx.handle, C.c_void_p(sh), Ls, stats))
        if Ls <= 64 and not args.no_diag:
            sets = []
            P = np.zeros(Dl, dtype=np.int32)
            V = np.zeros(Dl, dtype=np.int32)
            p, v = C.c_int64(0), C.c_int64(0)
            for l in range(Ls):
                check(lib.sg_ctx_read_stack_sets(ctx.handle, C.c_void_p(sh), l,
                                                 P.ctypes.data_as(C.c_void_p), C.byref(p),
                                                 V.ctypes.data_as(C.c_void_p), C.byref(v)))
                sets.append((P[:p.value].astype(np.int64), V[:v.value].astype(np.int64)))
            check(lib.sg_ctx_enable_stack_sets(ctx.handle, 0))
    elif sharded:
        step_layers()
        check(lib.sg_ctx_read_stack_stats(ctx.handle, C.c_void_p(sh), Ls, stats))
    else:
        for l in range(Ls):
            src = ys[l - 1] if (chain == 1 and l > 0) else xs[l]
            layers[l].forward_device(src.data_ptr(), ys[l].data_ptr(), Pipeline.Sequential, ctx, sh)
            s1 = capi.sg_exec_stats()
            check(lib.sg_ctx_read_stats(ctx.handle, C.c_void_p(sh), C.byref(s1)))
            stats[l] = s1
    ps = [int(s.predicted_active) for s in stats]
    vs = [int(s.revalidated) for s in stats]
    alg_bytes = sum(touched_bytes(d, Dl, args.rank, p, v) for p, v in zip(ps, vs))
    hbm, hbm_kind = peaks()
    per_launch_ms = ms / launches_per_step
    achieved = alg_bytes / launches_per_step / (per_launch_ms * 1e-3) / 1e9
    diag = None
    if sets is not None and world == 1 and Dl == D:
        xin = [xs[0].double().cpu().numpy()] + \
              [({0: xs[l], 1: ys[l - 1], 2: xs[l] + ys[l - 1]}[chain]).double().cpu().numpy()
               for l in range(1, Ls)]
        diag = near_threshold(host_l, None, xin, sets, cfg["act"])

    # e2e through the C ABI host entry: pinned x in, y out, synchronised per step
    xh = torch.empty((Ls, d), dtype=torch.float32, pin_memory=True)
    xh.copy_(xs.cpu())
    yh = torch.empty((Ls, d), dtype=torch.float32, pin_memory=True)

    def step_e2e():
        check(lib.sg_ffn_forward_layers_host(ctx.handle, arr, Ls, int(Pipeline.Sequential),
                                             C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()),
                                             chain, None, C.c_void_p(sh)))

    def step_e2e_sharded():
        # same call shape with the per-layer NCCL exchange: pinned x in, full y out
        xs.copy_(xh, non_blocking=True)
        step_layers()
        yh.copy_(ys, non_blocking=True)
        stream.synchronize()

    ke = max(10, min(args.steps, 500))
    ms_e2e, _ = timed(step_e2e if not sharded else step_e2e_sharded, ke, 3)
    h2d = (d if chain == 1 else Ls * d) * 4
    e2e = {"value": 1000.0 * copies / ms_e2e if copies > 1 else 1000.0 / ms_e2e, "unit": "tokens/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": Ls * d * 4, "ms_per_step": ms_e2e,
           "steps": ke,
           "call": "sg_ffn_forward_layers_host" if not sharded else
                   "H2D + sg_ffn_forward_layers_sharded (launches + NCCL all-reduces from C++) + D2H"}

    dense = None
    if not args.no_dense:
        ms_dense, _ = timed(lambda: step_stack(Pipeline.Dense) if is_stack else
                            step_layers(Pipeline.Dense), max(10, args.steps // 4), 3)
        dense = {"ms_per_step": ms_dense, "tokens_per_s": 1000.0 * (copies if copies > 1 else 1) / ms_dense,
                 "per_layer_us": ms_dense * 1000.0 / Ls,
                 "achieved_gbs": dense_bytes(d, Dl) * Ls / (ms_dense * 1e-3) / 1e9,
                 "sparse_speedup": ms_dense / ms}

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            meta = tj.get("_meta", {}).get(args.config)
            if meta and Dl == D:  # ncu DRAM bytes per layer x layers per launch of this run
                traffic = meta["per_layer"] * (Ls / launches_per_step)
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_for(cfg, host[0], args)
        except Exception as e:  # report, never fake
            cpu = {"value": None, "error": str(e)[:200]}

    if rank == 0:
        # tokens/s: one decode token through the L-layer model per step (for configs[0],
        # 4 rotated copies of the one layer per launch = 4 tokens)
        tok_s = 1000.0 * copies / ms if copies > 1 else 1000.0 / ms
        conf = bench_config(cfg, args, L, world)
        conf.update({
            "l2": ("no flush: each step streams %.2f GB of distinct layers (> 126 MB L2)" % (alg_bytes / 1e9))
                  if copies == 1 else
                  "no flush: each launch rotates over 4 device copies of the layer "
                  "(%.0f MB touched > 126 MB L2)" % (alg_bytes / 1e6),
            "predictor": "naive-mode randomized rank-r SVD + greedy calibration (eta 8)",
            "layout": "ascending" if args.no_balance else
                      "per-CTA load-balanced neuron order from calibration statistics",
            "hot_rows": 0 if args.no_balance else args.hot_rows,
            "mode": "stack (one persistent launch per step)" if is_stack else
                    ("C++ sharded step: per-layer launches + one NCCL all-reduce per layer "
                     "(sg_ffn_forward_layers_sharded)" if sharded else "per-layer launches"),
            "graph": graph_mode})
        line = {
            "metric": "sparse-FFN decode tokens/s", "value": tok_s, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": conf,
            "per_layer_us": ms * 1000.0 / Ls,
            "p_mean": float(np.mean(ps)), "v_mean": float(np.mean(vs)),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_kind": hbm_kind,
                         "frac_of_8000_nominal": achieved / 8000.0,
                         "traffic": traffic,
                         "bytes_per_launch": alg_bytes / launches_per_step,
                         "kernel": "ffn_kernel<2> (sequential executor)"},
            "unchained": unchained,
            "near_threshold": diag,
            "dense": dense,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        lib.sg_comm_destroy(comm)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
