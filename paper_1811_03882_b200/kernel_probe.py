"""Compile-probe backend for the reference's ExternalOracle on B200.

The reference decides a loop's eligibility either with built-in rules or by
handing a compiler the program with ONE `#pragma acc kernels` line in front
of the candidate loop (`ExternalOracle`, reference `analysis.py:181-216`;
paper §4: "does the loop compile to a kernel").  On B200 the question is
"does this loop map to one of our sm_100a kernels, does the launcher accept
its shape, and does that kernel build for sm_100a".  This module answers it
as a command the reference interface can run unchanged:

    --oracle cmd:probe.json   with   {"compile_cmd":
        "python -m paper_1811_03882_b200.kernel_probe {src}"}

Exit status 0 = eligible.  Steps:

1. find the loop after the `#pragma acc kernels` line and recognise it as a
   Darknet op: the loop text must equal, line for line, what the op emitter
   (`nets._emit_op`) writes for the kind and shape read off its headers;
2. check the shape against the kernel launcher's preconditions (the same
   32-bit / grid limits `acct_*_f32` enforce: ACCT_EINVAL / ACCT_ENOTSUP);
3. trial-build the product's kernel source for the launch configuration the
   runtime would pick (`nvcc -gencode arch=compute_100a,code=sm_100a -cubin`
   of a unit that includes the implementing .cu and takes the address of that
   template instance) and check the cubin holds the kernel -- and, for the
   tensor-core gemm, tcgen05 MMAs (SASS `UTCHMMA`).

Builds are cached by (kernel source hash, instance) under
`$ACCT_PROBE_CACHE` (default `paper_1811_03882_b200/.probe_cache`).
"""

from __future__ import annotations

import hashlib
import os
import re
import subprocess
import sys
import tempfile
from dataclasses import dataclass
from pathlib import Path

from . import nets

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
HEADER = re.compile(r"^for \((\w+) = 0; \1 < (\d+); \1\+\+\) \{$")


@dataclass
class Probe:
    eligible: bool
    reason: str
    kind: str | None = None
    params: dict | None = None
    instance: str | None = None


# ------------------------------------------------------------ recognition
def candidate_block(source: str) -> list[str] | None:
    """The candidate loop's lines (dedented) after the kernels pragma."""
    lines = source.splitlines()
    at = next((i for i, line in enumerate(lines) if line.strip() == "#pragma acc kernels"), None)
    if at is None or at + 1 >= len(lines):
        return None
    head = lines[at + 1]
    indent = len(head) - len(head.lstrip())
    if not head.strip().startswith("for ("):
        return None
    depth, out = 0, []
    for line in lines[at + 1:]:
        out.append(line[indent:] if line[:indent].strip() == "" else line.strip())
        depth += line.count("{") - line.count("}")
        if depth == 0:
            return out
    return None


def _headers(block: list[str]) -> list[tuple[str, int]]:
    """(var, trip) of the leading perfectly nested loop headers."""
    out = []
    for line in block:
        m = HEADER.match(line.strip())
        if not m:
            break
        out.append((m.group(1), int(m.group(2))))
    return out


def _emit(kind: str, arrays: dict, params: dict) -> list[str]:
    w = nets._Writer()
    nets._emit_op(w, nets.OpSpec(kind, 0, arrays=arrays, params=params))
    return w.lines


def recognize(block: list[str]) -> tuple[str, dict, dict] | None:
    """(kind, params, arrays) if the block is exactly one emitted Darknet op."""
    hs = _headers(block)
    body = " ".join(line.strip() for line in block)
    ident = r"([A-Za-z_]\w*)"
    guesses: list[tuple[str, dict, dict]] = []
    if [v for v, _ in hs[:2]] == ["i", "j"] and len(hs) == 2:
        M, N = hs[0][1], hs[1][1]
        p = {"M": M, "N": N}
        m = re.search(ident + r"\[i\]\[j \* 1\] = 0\.0;", body)
        if m:
            guesses.append(("fill", p, {"Y": m.group(1)}))
        m = re.search(ident + r"\[i\]\[j \* 1\] \+= " + ident + r"\[i\];", body)
        if m:
            guesses.append(("add_bias", p, {"Y": m.group(1), "bias": m.group(2)}))
        m = re.search(r"if \(" + ident + r"\[i\]\[j \* 1\] < 0\.0\)", body)
        if m:
            guesses.append(("leaky", p, {"Y": m.group(1)}))
        m = re.search(ident + r"\[i\]\[j \* 1\] = " + ident + r"\[i\]\[j \* 1\];", body)
        if m:
            kind = "linear" if m.group(1) == m.group(2) else "copy"
            arrays = {"Y": m.group(1)} if kind == "linear" else {"Y": m.group(1), "X": m.group(2)}
            guesses.append((kind, p, arrays))
    if [v for v, _ in hs] == ["i", "k", "j"]:
        m = re.search(ident + r"\[i\]\[j \* 1\] \+= " + ident + r"\[i\]\[k\] \* " + ident
                      + r"\[k\]\[j \* 1\];", body)
        if m:
            guesses.append(("gemm", {"M": hs[0][1], "K": hs[1][1], "N": hs[2][1]},
                            {"C": m.group(1), "A": m.group(2), "B": m.group(3)}))
    if [v for v, _ in hs] == ["c", "h", "w"]:
        m = re.search(r"if \(c / (\d+) % \1 \+ h \* (\d+) - (\d+) < 0 \|\| .* >= (\d+) \|\| "
                      r"c % \1 \+ w \* \2 - \3 < 0 \|\| .* >= (\d+)\) \{ " + ident
                      + r"\[c\]\[h \* (\d+) \+ w\] = 0\.0; \} else \{ \6\[c\]\[h \* \7 \+ w\] = "
                      + ident + r"\[c / (\d+)\]", body)
        if m:
            k, s, pad, H, W = (int(m.group(i)) for i in range(1, 6))
            K, oh, ow = hs[0][1], hs[1][1], hs[2][1]
            if k > 0 and K % (k * k) == 0:
                guesses.append(("im2col", {"c": K // (k * k), "h": H, "w": W, "ksize": k,
                                           "stride": s, "pad": pad, "oh": oh, "ow": ow,
                                           "K": K, "N": oh * ow},
                                {"X": m.group(8), "Y": m.group(6)}))
    if [v for v, _ in hs] == ["c", "i", "j"]:
        m = re.search(ident + r"\[c\]\[i \* (\d+) \+ j\] = -[0-9.e+]+; " + ident
                      + r"\[c\]\[i \* \2 \+ j\] = -1; for \(n = 0; n < (\d+); n\+\+\) \{ .*?"
                      r"if \(i \* (\d+) \+ n - (\d+) >= 0 && i \* \5 \+ n - \6 < (\d+) && "
                      r"j \* \5 \+ m - \6 >= 0 && j \* \5 \+ m - \6 < (\d+)\) \{ if \("
                      + ident + r"\[c\]", body)
        if m:
            guesses.append(("maxpool", {"c": hs[0][1], "h": int(m.group(7)),
                                        "w": int(m.group(8)), "size": int(m.group(4)),
                                        "stride": int(m.group(5)), "off": int(m.group(6)),
                                        "oh": hs[1][1], "ow": hs[2][1]},
                            {"X": m.group(9), "Y": m.group(1), "I": m.group(3)}))
    want = [line.rstrip() for line in block]
    for kind, params, arrays in guesses:
        if [line.rstrip() for line in _emit(kind, arrays, params)] == want:
            return kind, params, arrays
    return None


# ------------------------------------------------------------ launch config
MAX_ELEMS = 1 << 31


def _pitch(n: int) -> int:
    from .executor import _pitch as executor_pitch   # the executor's device row pitch
    return executor_pitch(n)


def launch_instance(kind: str, p: dict) -> tuple[str | None, str, str]:
    """(kernel source file, C++ expression naming the template instance the
    runtime launches, reason) -- source None = no device work (identity)."""
    if kind in ("fill", "copy", "add_bias", "leaky"):
        op = {"fill": 0, "copy": 1, "add_bias": 2, "leaky": 3}[kind]
        if p["M"] > 65535 * 8 or p["M"] * _pitch(p["N"]) >= MAX_ELEMS:
            raise ValueError("rows x pitch beyond 32-bit indexing (ACCT_ENOTSUP)")
        return "acct_elementwise.cu", f"rows_vec<{op}>", "2-D float4 sweep"
    if kind == "linear":
        return None, "", "identity loop: no device work (ACCT_ACT_LINEAR)"
    if kind == "im2col":
        if p["K"] > 65535 or p["K"] * _pitch(p["N"]) >= MAX_ELEMS:
            raise ValueError("im2col too large for 32-bit indexing (ACCT_ENOTSUP)")
        if p["ksize"] == 3 and p["stride"] == 1 and p["pad"] == 1:
            if 16 <= p["ow"] < 64:
                return "acct_elementwise.cu", "im2col_k3s1_flat_kernel", "3x3/1/1 pixel kernel"
            return "acct_elementwise.cu", "im2col_k3s1_kernel", "3x3/1/1 window kernel"
        if p["ow"] >= 64:
            return "acct_elementwise.cu", "im2col_rows_kernel", "row kernel"
        return "acct_elementwise.cu", "im2col_kernel", "flat kernel"
    if kind == "maxpool":
        if p["c"] > 65535 or p["c"] * _pitch(p["h"] * p["w"]) >= MAX_ELEMS:
            raise ValueError("maxpool too large for 32-bit indexing (ACCT_ENOTSUP)")
        if (p["size"] == 2 and p["stride"] == 2 and p["off"] == 0 and p["h"] == 2 * p["oh"]
                and p["w"] == 2 * p["ow"] and p["ow"] % 2 == 0 and p["w"] % 4 == 0):
            v = 4 if p["ow"] % 4 == 0 else 2
            return "acct_elementwise.cu", f"maxpool2s2_kernel<{v}>", "2x2/2 vector kernel"
        if p["ow"] >= 32:
            return "acct_elementwise.cu", "maxpool_rows_kernel", "row kernel"
        return "acct_elementwise.cu", "maxpool_kernel", "flat kernel"
    if kind == "gemm":
        M, N, K = p["M"], p["N"], p["K"]
        if K * 32 * 4 <= 200 * 1024 and (M <= 16 or (M <= 32 and K <= 64)):
            inst = "gemm_stream_kernel<16, 8>" if M <= 16 else "gemm_stream2_kernel<32, 8>"
            return "acct_gemm_simt.cu", inst, "HBM-streaming FP32 kernel"
        if M <= 32:
            return "acct_gemm_tc.cu", "acct::tc_gemm_kernel<32, true, 32>", "tcgen05 swap tile"
        if M <= 64:
            return "acct_gemm_tc.cu", "acct::tc_gemm_kernel<64, true, 32>", "tcgen05 swap tile"
        choice = gemm_tile(M, N, K)
        if choice == "pair256":
            return ("acct_gemm_tc.cu", "acct::tc2_gemm_kernel<256, 1, 32, false>",
                    "tcgen05 CTA-pair 256x256 tile (cta_group::2)")
        if choice == "pair192":
            return ("acct_gemm_tc.cu", "acct::tc2_gemm_kernel<192, 1, 32, false>",
                    "tcgen05 CTA-pair 256x192 tile (cta_group::2)")
        return ("acct_gemm_tc.cu", "acct::tc_gemm_kernel<192, false, 16>",
                "tcgen05 128x192 tile (operand A in TMEM)")
    raise KeyError(kind)


# the tile choice of gemm_tc (acct_gemm_tc.cu), restated for the probe
SMS = 148


def _plan_splits(tiles: int, total_kb: int, sms: int) -> tuple[int, int]:
    splits = 1
    if tiles < sms:
        splits = max(1, min(sms // tiles, total_kb // 2))
    kb_per = -(-total_kb // splits)
    return -(-total_kb // kb_per), kb_per


def _cost(M: int, N: int, K: int, tn: int, bk: int, rows: int, units: int) -> int:
    tiles = -(-M // rows) * -(-N // tn)
    splits, kb_per = _plan_splits(tiles, -(-K // bk), units)
    return -(-(tiles * splits) // units) * kb_per * bk * tn


def gemm_tile(M: int, N: int, K: int, sms: int = SMS) -> str:
    c1 = 1.25 * _cost(M, N, K, 192, 16, 128, sms)
    waste = (-(-M // 256) * 256) / (-(-M // 128) * 128)
    c9 = waste * _cost(M, N, K, 192, 32, 256, sms // 2)
    c10 = waste * _cost(M, N, K, 256, 32, 256, sms // 2)
    if c10 < c9 and c10 < c1:
        return "pair256"
    return "pair192" if c9 < c1 else "single192"


# ------------------------------------------------------------ trial build
def cache_dir() -> Path:
    d = Path(os.environ.get("ACCT_PROBE_CACHE", PKG / ".probe_cache"))
    d.mkdir(parents=True, exist_ok=True)
    return d


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def trial_build(source: str, instance: str) -> tuple[bool, str]:
    """nvcc the implementing kernel source for sm_100a with `instance`
    referenced; the cubin must contain that kernel (and UTCHMMA for tcgen05)."""
    src = CSRC / source
    key_text = src.read_text() + instance + (CSRC / "acct_common.cuh").read_text() + \
        (CSRC / "acct_tc.cuh").read_text()
    key = hashlib.sha256(key_text.encode()).hexdigest()[:20]
    stamp = cache_dir() / f"{key}.ok"
    if stamp.exists():
        return True, stamp.read_text()
    with tempfile.TemporaryDirectory(prefix="acct_probe_") as tmp:
        unit = Path(tmp) / "trial.cu"
        unit.write_text(f'#include "{src}"\n'
                        f"void *acct_probe_instance = (void *)&{instance};\n")
        cubin = Path(tmp) / "trial.cubin"
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-w",
               "-cubin", "-I", str(INCLUDE), "-I", str(CSRC), "-o", str(cubin), str(unit)]
        done = subprocess.run(cmd, capture_output=True, text=True)
        if done.returncode != 0:
            return False, "nvcc failed: " + done.stderr.strip().splitlines()[-1:][0] \
                if done.stderr.strip() else "nvcc failed"
        sass = subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True,
                              text=True).stdout
        base = instance.split("::")[-1].split("<")[0]
        if base not in sass:
            return False, f"kernel {base} missing from the sm_100a cubin"
        if "gemm_kernel<" in instance and "tc" in instance and "UTCHMMA" not in sass:
            return False, "no tcgen05 MMA (UTCHMMA) in the tensor-core kernel"
        tc = "tc_gemm" in instance or "tc2_gemm" in instance
        note = f"sm_100a cubin with {base}" + (" (UTCHMMA)" if tc else "")
    stamp.write_text(note)
    return True, note


def probe_source(source: str, build: bool = True) -> Probe:
    block = candidate_block(source)
    if block is None:
        return Probe(False, "no '#pragma acc kernels' followed by a for loop")
    hit = recognize(block)
    if hit is None:
        return Probe(False, "loop is not a Darknet op this backend has a kernel for")
    kind, params, _ = hit
    try:
        file, instance, why = launch_instance(kind, params)
    except ValueError as exc:
        return Probe(False, f"{kind}: {exc}", kind, params)
    if file is None:
        return Probe(True, f"{kind}: {why}", kind, params)
    if not build:
        return Probe(True, f"{kind}: {instance} ({why}); build skipped", kind, params, instance)
    ok, note = trial_build(file, instance)
    return Probe(ok, f"{kind}: {instance} ({why}): {note}", kind, params, instance)


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) != 1:
        print("usage: python -m paper_1811_03882_b200.kernel_probe <trial.c>", file=sys.stderr)
        return 2
    res = probe_source(Path(argv[0]).read_text())
    print(("eligible: " if res.eligible else "rejected: ") + res.reason, file=sys.stderr)
    return 0 if res.eligible else 1


if __name__ == "__main__":
    sys.exit(main())
