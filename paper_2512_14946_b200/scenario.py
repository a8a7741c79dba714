"""Scenario ingestion: the reference's scenario files
(proj/src/workload.cpp:467-618 `load_scenario_text` / `load_scenario_file`)
read straight into the serve loop's `Scenario` + trace, so
`serve.Replayer` runs the reference's own scenario files: tiers, params,
methods / ratio grid, profiles (inline, JSONL file, or generated from dataset
presets / custom blocks, with drifted truth curves), traces (inline, JSONL
file, or generated: Poisson arrivals over Zipf popularity, popularity-matched
frequencies), dotted-path overrides, drift settings. Generators reproduce
the reference's RNG streams bit for bit (std::mt19937_64 through
`serve.MT19937_64`, the same Box-Muller / log1p / pow transforms from the
same libm).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from . import _abi as A
from .kvtier import CandidateSpace, CompressionMethod, ContextProfile, TierSpec, UtilityParams
from .serve import GRID_EPS, MT19937_64, Request, Scenario, synth_quality

_MASK = (1 << 64) - 1
K_BLOCK, K_TRACE, K_SHUFFLE, K_DRIFT = 0xB10C, 0x7ACE, 0x54F1, 0xD21F  # workload.cpp:32-35
K_MIN_TOKENS, K_MAX_TOKENS = 1e3, 2e5  # workload.hpp:37-38
DEFAULT_METHODS = ("keydiff", "knorm", "snapkv")
DEFAULT_GRID = (0.05, 0.1, 0.2, 0.4, 0.6, 0.8, 0.9, 1.0)
# workload.cpp:112-127: name, mean tokens, std tokens, has sensitivity, median sensitivity
PRESETS = {p[0]: p for p in [
    ("narrativeqa", 108e3, 55e3, True, 0.340), ("qasper", 24e3, 12e3, True, 0.759),
    ("multifieldqa_en", 29e3, 15e3, False, 0.0), ("hotpotqa", 57e3, 18e3, False, 0.0),
    ("2wikimqa", 30e3, 15e3, True, 0.681), ("musique", 69e3, 9e3, False, 0.0),
    ("gov_report", 54e3, 34e3, False, 0.0), ("qmsum", 57e3, 27e3, False, 0.0),
    ("multi_news", 12e3, 10e3, True, 0.738), ("trec", 30e3, 12e3, False, 0.0),
    ("triviaqa", 47e3, 25e3, True, 0.392), ("samsum", 34e3, 17e3, True, 0.676)]}


def _err(msg):
    return A.ValidationError(A.KVT_EVALIDATION, msg)


def mix64(seed: int, stream: int) -> int:  # workload.cpp:21-29
    x = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & _MASK
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _MASK
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _MASK
    x ^= x >> 31
    return x


class Rng(MT19937_64):  # proj/include/kvtier/rng.hpp
    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def normal(self, mean: float, stddev: float) -> float:
        u1, u2 = self.uniform01(), self.uniform01()
        while u1 <= 0.0:
            u1 = self.uniform01()
        radius = math.sqrt(-2.0 * math.log(u1))
        return mean + stddev * radius * math.cos(2.0 * math.pi * u2)

    def truncated_normal(self, mean: float, stddev: float, lo: float, hi: float) -> float:
        if stddev <= 0.0:
            return min(max(mean, lo), hi)
        while True:
            x = self.normal(mean, stddev)
            if lo <= x <= hi:
                return x

    def exponential(self, rate: float) -> float:
        return -math.log1p(-self.uniform01()) / rate

    def uniform_index(self, n: int) -> int:
        return self.next_u64() % n


class Zipf:  # rng.hpp ZipfSampler
    def __init__(self, n: int, exponent: float):
        cdf, total = [], 0.0
        for i in range(n):
            total += math.pow(float(i + 1), -exponent)
            cdf.append(total)
        self.cdf = [c / total for c in cdf]

    def sample(self, rng: Rng) -> int:
        u = rng.uniform01()
        lo, hi = 0, len(self.cdf) - 1
        while lo < hi:
            mid = (lo + hi) // 2
            if self.cdf[mid] < u:
                lo = mid + 1
            else:
                hi = mid
        return lo

    def weight(self, rank: int) -> float:
        return self.cdf[0] if rank == 0 else self.cdf[rank] - self.cdf[rank - 1]


@dataclass
class SensDist:  # quality.hpp SensitivityDist
    kind: str
    median: float = 0.0
    cov: float = 0.0
    lo: float = 0.0
    hi: float = 1.0
    shape_k: float = 1.0

    def draw(self, rng: Rng) -> float:  # quality.cpp draw_sensitivity
        s = rng.uniform(self.lo, self.hi) if self.kind == "uniform" else rng.normal(self.median, self.cov * self.median)
        return min(max(s, 0.0), 1.0)


def parse_sensitivity(j: dict, default_k: float) -> SensDist:  # workload.cpp:336-348
    kind = j.get("kind", "normal")
    k = float(j.get("shape_k", default_k))
    if kind == "normal":
        return SensDist("normal", median=float(j["median"]), cov=float(j.get("cov", 0.2)), shape_k=k)
    if kind == "uniform":
        return SensDist("uniform", lo=float(j.get("lo", 0.0)), hi=float(j.get("hi", 1.0)), shape_k=k)
    raise _err(f"unknown sensitivity kind '{kind}' (expected normal or uniform)")


def gen_profiles(seed: int, n: int, prefix: str, sens: Dict[str, SensDist], mean_size: float, std_size: float,
                 min_size: float, max_size: float, frequency: float, grid: List[float]):
    """quality.cpp gen_profiles: (profiles, truth curves) for n contexts."""
    if max_size <= 0.0:
        max_size = mean_size + 10.0 * std_size
    rng = Rng(seed)
    digits = len(str(n - 1)) if n > 0 else 1
    out = []
    for i in range(n):
        cid = "%s-%0*d" % (prefix, digits, i)
        size = rng.truncated_normal(mean_size, std_size, min_size, max_size)
        table, truth = {}, {}
        for m in sorted(sens, key=lambda x: x.encode()):  # std::map order
            d = sens[m]
            s = d.draw(rng)
            truth[m] = (s, d.shape_k)
            table[m] = [synth_quality(s, d.shape_k, r) for r in grid]
        out.append((ContextProfile(cid, max(1, int(size)), frequency, list(grid), table), truth))
    return out


def gen_contexts(seed: int, block: dict, params: UtilityParams, methods: Sequence[str], grid: Sequence[float]):
    """workload.cpp:152-212 (one profiles.generate block)."""
    k = float(block.get("shape_k", 1.0))
    cov = float(block.get("cov", 0.2))
    mean_tokens = float(block.get("mean_tokens", 0.0))
    std_tokens = float(block.get("std_tokens", -1.0))
    prefix = block.get("id_prefix", "")
    sens = parse_sensitivity(block["sensitivity"], k) if "sensitivity" in block else None
    drifted = parse_sensitivity(block["drifted_sensitivity"], k) if "drifted_sensitivity" in block else None
    preset = block.get("preset", "")
    if preset:
        if preset not in PRESETS:
            raise _err(f"unknown dataset preset '{preset}' (available: {', '.join(PRESETS)})")
        _, pm, ps, has, med = PRESETS[preset]
        if mean_tokens <= 0.0:
            mean_tokens = pm
        if std_tokens < 0.0:
            std_tokens = ps
        if sens is None:
            sens = SensDist("normal", median=med, cov=cov, shape_k=k) if has else SensDist("uniform", shape_k=k)
        if not prefix:
            prefix = preset
    else:
        if mean_tokens <= 0.0:
            raise _err("custom context block needs mean_tokens > 0")
        std_tokens = max(std_tokens, 0.0)
        if sens is None:
            sens = SensDist("uniform", shape_k=k)
        if not prefix:
            prefix = "ctx"
    g = sorted(set(float(x) for x in grid))
    out = gen_profiles(seed, int(block.get("n", 0)), prefix, {m: sens for m in methods},
                       mean_tokens * params.bytes_per_token, std_tokens * params.bytes_per_token,
                       K_MIN_TOKENS * params.bytes_per_token, K_MAX_TOKENS * params.bytes_per_token,
                       float(block.get("frequency", 1.0)), g)
    if drifted is not None:  # the world's truth drifts away from the profiled curves
        rng = Rng(mix64(seed, K_DRIFT))
        for _, truth in out:
            for m in methods:
                truth[m] = (drifted.draw(rng), drifted.shape_k)
    return out


def _ranks(seed: int, n: int, shuffle: bool) -> List[int]:  # workload.cpp:63-76
    rank = list(range(n))
    if shuffle and n > 1:
        rng = Rng(mix64(seed, K_SHUFFLE))
        for i in range(n, 1, -1):
            j = rng.uniform_index(i)
            rank[i - 1], rank[j] = rank[j], rank[i - 1]
    return rank


def _trace_gen(j: dict):  # workload.cpp:415-423 (+ validate_trace_gen)
    p = {"arrival_rate": float(j.get("arrival_rate", 1.0)), "duration": float(j.get("duration", 0.0)),
         "zipf_exponent": float(j.get("zipf_exponent", 1.0)), "n_new_tokens": int(j.get("n_new_tokens", 0)),
         "shuffle_ranks": bool(j.get("shuffle_ranks", True))}
    if not p["arrival_rate"] > 0.0:
        raise _err("trace arrival_rate must be > 0")
    if not p["duration"] > 0.0:
        raise _err("trace duration must be > 0")
    if p["zipf_exponent"] < 0.0:
        raise _err("zipf_exponent must be >= 0")
    if p["n_new_tokens"] < 0:
        raise _err("n_new_tokens must be >= 0")
    return p


def gen_trace(seed: int, ids: List[str], p: dict) -> List[Request]:  # workload.cpp:214-232
    rank = _ranks(seed, len(ids), p["shuffle_ranks"])
    ctx_of_rank = [0] * len(ids)
    for i, r in enumerate(rank):
        ctx_of_rank[r] = i
    rng = Rng(seed)
    zipf = Zipf(len(ids), p["zipf_exponent"])
    out, t = [], 0.0
    while True:
        t += rng.exponential(p["arrival_rate"])
        if t > p["duration"]:
            break
        out.append(Request(t, ids[ctx_of_rank[zipf.sample(rng)]], p["n_new_tokens"]))
    return out


def _profile_from_json(j: dict):  # quality.cpp:327-370
    cid = j["context_id"]
    grid = [float(x) for x in j["grid"]]
    table = {}
    for m, row in j["methods"].items():
        vals = [-1.0] * len(grid)
        for rt, q in row.items():
            r = float(rt)
            hit = [i for i, g in enumerate(grid) if abs(g - r) <= GRID_EPS]
            if not hit:
                raise A.AbiError(A.KVT_ETRACE, f"profile ratio {rt} not on grid for context {cid}")
            vals[hit[0]] = float(q)
        if any(v < 0.0 for v in vals):
            raise A.AbiError(A.KVT_ETRACE, f"method {m} missing a grid ratio for context {cid}")
        table[m] = vals
    truth = {m: (float(c["s"]), float(c["k"])) for m, c in j.get("truth", {}).items()}
    return ContextProfile(cid, int(j["size_bytes"]), float(j.get("frequency", 1.0)), grid, table), truth


def _request(j: dict) -> Request:  # workload.cpp:78-93
    r = Request(float(j["t"]), j["context_id"], int(j.get("n_new_tokens", 0)))
    if not r.context or not math.isfinite(r.t) or r.n_new_tokens < 0:
        raise A.AbiError(A.KVT_ETRACE, f"bad trace request {j}")
    return r


def _jsonl(path: str) -> List[dict]:
    with open(path) as f:
        return [json.loads(line) for line in f if line.strip()]


def apply_override(doc: dict, assignment: str):  # workload.cpp:439-490
    if "=" not in assignment or assignment.startswith("="):
        raise _err("override must look like path.to.key=value: " + assignment)
    path, text = assignment.split("=", 1)
    try:
        value = json.loads(text)
    except ValueError:
        value = text  # bare strings need no quotes
    keys = path.split(".")
    node = doc
    for i, key in enumerate(keys):
        if not key:
            raise _err("override has an empty path segment: " + assignment)
        last = i + 1 == len(keys)
        if key.isdigit() and isinstance(node, list):
            idx = int(key)
            if idx >= len(node):
                raise _err(f"override index {key} out of range in: {path}")
            if last:
                node[idx] = value
            else:
                node = node[idx]
        else:
            if not isinstance(node, dict):
                raise _err("override path crosses a non-object value: " + path)
            if last:
                node[key] = value
            else:
                if node.get(key) is None:
                    node[key] = {}
                node = node[key]


def load_scenario_text(text: str, base_dir: str = "",
                       overrides: Sequence[str] = ()) -> Tuple[Scenario, List[Request], str]:
    """workload.cpp:492-612 -> (Scenario, trace, policy label)."""
    doc = json.loads(text)
    for o in overrides:
        apply_override(doc, o)
    seed = int(doc.get("seed", 0)) & _MASK
    pj = doc.get("params", {})
    params = UtilityParams(float(pj.get("alpha", 1.0)), float(pj.get("prefill_a", 2e-5)),
                           float(pj.get("prefill_b", 1e-10)), float(pj.get("bytes_per_token", 1.2e5)))
    if "alpha" in doc:
        params.alpha = float(doc["alpha"])
    if "methods" in doc:
        methods = [CompressionMethod(m, 0.0) if isinstance(m, str) else
                   CompressionMethod(m["name"], float(m.get("decompression_overhead", 0.0))) for m in doc["methods"]]
    else:
        methods = [CompressionMethod(m, 0.0) for m in DEFAULT_METHODS]
    grid = [float(x) for x in doc.get("ratio_grid", DEFAULT_GRID)]
    space = CandidateSpace(methods, grid)
    if not isinstance(doc.get("tiers"), list) or not doc["tiers"]:
        raise _err("scenario needs a non-empty tiers array")
    tiers = []
    for index, t in enumerate(doc["tiers"]):  # workload.cpp:383-413
        tid = int(t.get("tier_id", index))
        cap = None
        if t.get("capacity_bytes") is not None:
            cap = int(_llround(float(t["capacity_bytes"])))
        elif t.get("capacity_gb") is not None:
            cap = int(_llround(float(t["capacity_gb"]) * 1e9))
        if "read_bandwidth" in t:
            bw = float(t["read_bandwidth"])
        elif "read_bandwidth_gbps" in t:
            bw = float(t["read_bandwidth_gbps"]) * 1e9
        else:
            raise _err(f"tier {t.get('name', tid)} needs read_bandwidth or read_bandwidth_gbps")
        tiers.append(TierSpec(tid, t.get("name", f"tier{tid}"), cap, bw, float(t.get("fixed_access_latency", 0.0))))
    tiers.sort(key=lambda x: x.tier_id)  # validate_hierarchy's stable order
    names = [m.name for m in methods]

    if "profiles" not in doc:
        raise _err("scenario needs a profiles section")
    prof = doc["profiles"]
    contexts: List[Tuple[ContextProfile, Dict[str, Tuple[float, float]]]] = []
    if "file" in prof:
        contexts = [_profile_from_json(j) for j in _jsonl(os.path.join(base_dir, prof["file"]))]
    elif "inline" in prof:
        contexts = [_profile_from_json(j) for j in prof["inline"]]
    elif "generate" in prof:
        for bi, block in enumerate(prof["generate"]):
            contexts += gen_contexts(mix64(seed, K_BLOCK + bi), block, params, names, grid)
    else:
        raise _err("profiles needs 'file', 'inline' or 'generate'")
    if not contexts:
        raise _err("scenario produced no contexts")

    if "trace" not in doc:
        raise _err("scenario needs a trace section")
    tr = doc["trace"]
    if "file" in tr or "inline" in tr:
        rows = _jsonl(os.path.join(base_dir, tr["file"])) if "file" in tr else tr["inline"]
        trace = [_request(j) for j in rows]
        if any(trace[i].t < trace[i - 1].t for i in range(1, len(trace))):
            trace.sort(key=lambda r: r.t)  # stable, like the reference's
    elif "generate" in tr:
        p = _trace_gen(tr["generate"])
        tseed = mix64(seed, K_TRACE)
        rank = _ranks(tseed, len(contexts), p["shuffle_ranks"])  # assign_zipf_frequencies
        zipf = Zipf(len(contexts), p["zipf_exponent"])
        for i, (cp, _) in enumerate(contexts):
            cp.frequency = p["arrival_rate"] * zipf.weight(rank[i])
        trace = gen_trace(tseed, [cp.context for cp, _ in contexts], p)
    else:
        raise _err("trace needs 'file', 'inline' or 'generate'")

    seen = set()
    for cp, _ in contexts:
        if cp.context in seen:
            raise _err("duplicate context id " + cp.context)
        seen.add(cp.context)
    for r in trace:
        if r.context not in seen:
            raise _err("trace references unknown context " + r.context)
    drift, dc = False, {}
    if "drift" in doc:  # workload.cpp:425-437
        d = doc["drift"]
        drift = bool(d.get("enabled", True))
        dc = {"threshold": float(d.get("threshold", 0.3)), "min_samples": int(d.get("min_samples", 10)),
              "window_size": int(d.get("window_size", 0)), "duration": float(d.get("duration", 2.0)),
              "penalty": float(d.get("penalty", 0.5)), "noise_amplitude": float(d.get("noise", 0.0)),
              "gpu_window": float(d.get("gpu_window", 1.0)), "max_batch": int(d.get("max_batch", 8))}
    policy = doc.get("policy", "joint")
    rule = "quality_first" if policy == "joint-qargmax" else "utility"
    sc = Scenario(tiers, params, space, [cp for cp, _ in contexts],
                  {cp.context: t for cp, t in contexts if t}, [cp.context for cp, _ in contexts],
                  bool(doc.get("warm_start", False)), bool(doc.get("miss_store_bottom", False)), drift, rule,
                  seed, dc, policy)
    return sc, trace, policy


def _llround(x: float) -> int:  # std::llround: nearest, half away from zero (x - floor(x) is exact)
    a = abs(x)
    f = math.floor(a)
    r = int(f) + (1 if a - f >= 0.5 else 0)
    return r if x >= 0 else -r


def load_scenario_file(path: str, overrides: Sequence[str] = ()) -> Tuple[Scenario, List[Request], str]:
    with open(path) as f:
        return load_scenario_text(f.read(), os.path.dirname(path), overrides)


__all__ = ["load_scenario_text", "load_scenario_file", "apply_override", "gen_contexts", "gen_trace", "mix64", "Rng",
           "Zipf"]
