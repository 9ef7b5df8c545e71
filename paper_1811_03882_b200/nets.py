"""Darknet-style CNN programs written in the reference's C subset.

The reference models Darknet only as a gene count (`PAPER.md:169`;
`pkg/tests/fixtures/generate.py:248-309`); the paper tuned the real
Darknet.  This module writes the network forward pass as a C-subset program
that the reference front end parses, analyses and plans exactly like any
other input, so the GA's genes are the CNN's loops:

    fill_cpu        out[i][j*1] = 0.0                       one gene per conv
    im2col_cpu      col[c][h*OW+w] = pad ? 0 : x[..]        (3x3 convs only)
    gemm_nn         out[i][j*1] += W[i][k] * col[k][j*1]    i-k-j, gene = i
    add_bias        out[i][j*1] += bias[i]
    activate        leaky: if (v < 0.0) v = 0.1 * v; linear: v = v
    forward_maxpool window max, strict '>', first max wins, -FLT_MAX pad,
                    argmax index written to an int array
    copy_cpu        y[i][j*1] = out[i][j*1]                 (region output)

Authoring rules that make exactly one gene per op:
arrays are 2-D `[channels][pixels]`; inner loops index the written array
through `j * 1` (unanalyzable, hence not genes); no scalar temporaries; all
arrays are parameters of `forward` (CPU-side defines, so their transfers can
hoist to the image loop).  The image loop `for (b ...)` calls
`load_input(x)` / `store_output(y)`; whole-array call arguments are CPU
ref+set, which is what pins `x` and `y` transfers inside the image loop.

`build_net(name)` returns a `NetProgram`: the source, per-array shapes, the
op manifest keyed by the op's gene loop id, the analytic loop profile and
the seeded synthetic data recipe.  Batch-norm is folded into the bias, as
the north star lists no normalize op.
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass, field

import numpy as np

FLT_MAX_LITERAL = "3.4028234663852886e+38"


@dataclass(frozen=True)
class Conv:
    filters: int
    size: int
    stride: int = 1
    activation: str = "leaky"       # leaky | linear


@dataclass(frozen=True)
class MaxPool:
    size: int
    stride: int


@dataclass(frozen=True)
class Region:
    """Darknet region layer output stage: a plain copy of its input."""


@dataclass(frozen=True)
class NetSpec:
    name: str
    channels: int
    height: int
    width: int
    layers: tuple
    images: int                     # trip count of the image loop


def _tiny_yolo_layers():
    L = []
    for f in (16, 32, 64, 128, 256):
        L += [Conv(f, 3), MaxPool(2, 2)]
    L += [Conv(512, 3), MaxPool(2, 1), Conv(1024, 3), Conv(512, 3),
          Conv(425, 1, activation="linear"), Region()]
    return tuple(L)


def _yolov2_layers():
    """yolov2.cfg layers 0-24 plus the 1024 3x3 and 425 1x1 heads, straight
    line (route/reorg omitted)."""
    L = [Conv(32, 3), MaxPool(2, 2), Conv(64, 3), MaxPool(2, 2),
         Conv(128, 3), Conv(64, 1), Conv(128, 3), MaxPool(2, 2),
         Conv(256, 3), Conv(128, 1), Conv(256, 3), MaxPool(2, 2),
         Conv(512, 3), Conv(256, 1), Conv(512, 3), Conv(256, 1), Conv(512, 3), MaxPool(2, 2),
         Conv(1024, 3), Conv(512, 1), Conv(1024, 3), Conv(512, 1), Conv(1024, 3),
         Conv(1024, 3), Conv(1024, 3),
         Conv(1024, 3), Conv(425, 1, activation="linear"), Region()]
    return tuple(L)


NETS = {
    # configs[0]: reference demo, conv16 3x3 + leaky + maxpool on 1x3x64x64
    "demo": NetSpec("demo", 3, 64, 64, (Conv(16, 3), MaxPool(2, 2)), images=8),
    # a tiny-YOLO-shaped net small enough for pure-Python parity tests
    "micro": NetSpec("micro", 3, 32, 32,
                     (Conv(8, 3), MaxPool(2, 2), Conv(16, 3), MaxPool(2, 1),
                      Conv(12, 1, activation="linear"), Region()), images=2),
    # configs[1]/[2]/[3]: yolov2-tiny 416x416, batch 1 per forward pass
    "yolov2-tiny": NetSpec("yolov2-tiny", 3, 416, 416, _tiny_yolo_layers(), images=16),
    # configs[4]: yolov2 608x608, batch 16
    "yolov2-608": NetSpec("yolov2-608", 3, 608, 608, _yolov2_layers(), images=16),
}


@dataclass
class ArraySpec:
    name: str
    dtype: str                      # 'float' | 'int'
    shape: tuple                    # (rows,) or (rows, cols)
    role: str                       # input | output | weight | bias | activation | workspace | index

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))

    @property
    def nbytes(self) -> int:
        return 4 * self.numel

    def decl(self) -> str:
        return f"{self.dtype} {self.name}" + "".join(f"[{d}]" for d in self.shape)


@dataclass
class OpSpec:
    kind: str                       # fill | im2col | gemm | add_bias | leaky | linear | maxpool | copy
    layer: int
    loop_id: int = -1               # the op's outer loop == its gene
    arrays: dict = field(default_factory=dict)   # role -> array name
    params: dict = field(default_factory=dict)   # int shape parameters

    def algorithmic_bytes(self) -> int:
        """Bytes a roofline-optimal implementation must move."""
        p = self.params
        if self.kind == "fill":
            return 4 * p["M"] * p["N"]
        if self.kind in ("copy", "leaky", "linear"):
            return 8 * p["M"] * p["N"]
        if self.kind == "add_bias":
            return 8 * p["M"] * p["N"] + 4 * p["M"]
        if self.kind == "im2col":
            return 4 * (p["K"] * p["N"] + p["c"] * p["h"] * p["w"])
        if self.kind == "maxpool":
            return 4 * (p["c"] * p["h"] * p["w"] + 2 * p["c"] * p["oh"] * p["ow"])
        if self.kind == "gemm":
            return 4 * (p["M"] * p["K"] + p["K"] * p["N"] + 2 * p["M"] * p["N"])
        raise KeyError(self.kind)

    def flops(self) -> int:
        return 2 * self.params["M"] * self.params["N"] * self.params["K"] if self.kind == "gemm" else 0


@dataclass
class NetProgram:
    spec: NetSpec
    source: str
    arrays: dict                    # name -> ArraySpec, in parameter order
    ops: list                       # OpSpec in program order
    loop_trips: list                # trip count per loop id
    loop_parent: list               # parent loop id per loop id (None for the image loop)
    image_loop: int
    input_name: str
    output_name: str

    @property
    def ops_by_loop(self) -> dict:
        return {op.loop_id: op for op in self.ops}

    def profile_dict(self) -> dict:
        rows = []
        for lid, trip in enumerate(self.loop_trips):
            entry = 1
            p = self.loop_parent[lid]
            while p is not None:
                entry *= self.loop_trips[p]
                p = self.loop_parent[p]
            rows.append({"id": lid, "entry_count": entry, "total_iterations": entry * trip})
        return {"loops": rows}

    def total_flops_per_image(self) -> int:
        return sum(op.flops() for op in self.ops)

    def total_bytes_per_image(self) -> int:
        return sum(op.algorithmic_bytes() for op in self.ops)


class _Writer:
    def __init__(self):
        self.lines: list[str] = []
        self.depth = 0
        self.trips: list[int] = []
        self.parents: list = []
        self.stack: list[int] = []

    def line(self, text: str):
        self.lines.append("    " * self.depth + text)

    def open_for(self, var: str, trip: int) -> int:
        lid = len(self.trips)
        self.trips.append(trip)
        self.parents.append(self.stack[-1] if self.stack else None)
        self.stack.append(lid)
        self.line(f"for ({var} = 0; {var} < {trip}; {var}++) {{")
        self.depth += 1
        return lid

    def close(self):
        self.depth -= 1
        self.line("}")
        self.stack.pop()

    def text(self) -> str:
        return "\n".join(self.lines) + "\n"


def build_net(name_or_spec, images: int | None = None) -> NetProgram:
    spec = NETS[name_or_spec] if isinstance(name_or_spec, str) else name_or_spec
    if images is not None:
        spec = NetSpec(spec.name, spec.channels, spec.height, spec.width, spec.layers, images)
    arrays: dict[str, ArraySpec] = {}

    def add(name, dtype, shape, role):
        arrays[name] = ArraySpec(name, dtype, tuple(shape), role)
        return name

    c, h, w = spec.channels, spec.height, spec.width
    cur = add("x", "float", (c, h * w), "input")
    ops: list[OpSpec] = []
    for li, layer in enumerate(spec.layers):
        if isinstance(layer, Conv):
            k, s = layer.size, layer.stride
            pad = k // 2
            oh = (h + 2 * pad - k) // s + 1
            ow = (w + 2 * pad - k) // s + 1
            M, K, N = layer.filters, c * k * k, oh * ow
            wt = add(f"w{li}", "float", (M, K), "weight")
            bias = add(f"bias{li}", "float", (M,), "bias")
            out = add(f"out{li}", "float", (M, N), "activation")
            ops.append(OpSpec("fill", li, arrays={"Y": out}, params={"M": M, "N": N}))
            if k == 1 and s == 1:
                operand = cur
            else:
                operand = add(f"col{li}", "float", (K, N), "workspace")
                ops.append(OpSpec("im2col", li, arrays={"X": cur, "Y": operand},
                                  params={"c": c, "h": h, "w": w, "ksize": k, "stride": s,
                                          "pad": pad, "oh": oh, "ow": ow, "K": K, "N": N}))
            ops.append(OpSpec("gemm", li, arrays={"A": wt, "B": operand, "C": out},
                              params={"M": M, "N": N, "K": K}))
            ops.append(OpSpec("add_bias", li, arrays={"Y": out, "bias": bias},
                              params={"M": M, "N": N}))
            ops.append(OpSpec(layer.activation, li, arrays={"Y": out}, params={"M": M, "N": N}))
            cur, c, h, w = out, M, oh, ow
        elif isinstance(layer, MaxPool):
            sz, st = layer.size, layer.stride
            padding = sz - 1                       # darknet default
            oh = (h + padding - sz) // st + 1
            ow = (w + padding - sz) // st + 1
            off = padding // 2                     # darknet: offset = -pad/2
            out = add(f"pool{li}", "float", (c, oh * ow), "activation")
            idx = add(f"idx{li}", "int", (c, oh * ow), "index")
            ops.append(OpSpec("maxpool", li, arrays={"X": cur, "Y": out, "I": idx},
                              params={"c": c, "h": h, "w": w, "size": sz, "stride": st,
                                      "off": off, "oh": oh, "ow": ow}))
            cur, h, w = out, oh, ow
        elif isinstance(layer, Region):
            out = add("y", "float", (c, h * w), "output")
            ops.append(OpSpec("copy", li, arrays={"X": cur, "Y": out},
                              params={"M": c, "N": h * w}))
            cur = out
        else:
            raise TypeError(layer)
    if not any(a.role == "output" for a in arrays.values()):
        arrays[cur].role = "output"
    output = next(a.name for a in arrays.values() if a.role == "output")

    W = _Writer()
    params = ", ".join(a.decl() for a in arrays.values())
    W.line(f"int forward({params}) {{")
    W.depth += 1
    W.line("int b; int i; int j; int k; int c; int h; int w; int n; int m;")
    image_loop = W.open_for("b", spec.images)
    W.line("load_input(x);")
    for op in ops:
        op.loop_id = len(W.trips)
        _emit_op(W, op)
    W.line(f"store_output({output});")
    W.close()
    W.line("return 0;")
    W.depth -= 1
    W.line("}")
    return NetProgram(spec, W.text(), arrays, ops, W.trips, W.parents, image_loop,
                      "x", output)


def _emit_op(W: _Writer, op: OpSpec):
    p, a = op.params, op.arrays
    if op.kind in ("fill", "add_bias", "leaky", "linear", "copy"):
        Y = a["Y"]
        W.open_for("i", p["M"])
        W.open_for("j", p["N"])
        if op.kind == "fill":
            W.line(f"{Y}[i][j * 1] = 0.0;")
        elif op.kind == "add_bias":
            W.line(f"{Y}[i][j * 1] += {a['bias']}[i];")
        elif op.kind == "leaky":
            W.line(f"if ({Y}[i][j * 1] < 0.0) {{ {Y}[i][j * 1] = 0.1 * {Y}[i][j * 1]; }}")
        elif op.kind == "linear":
            W.line(f"{Y}[i][j * 1] = {Y}[i][j * 1];")
        else:
            W.line(f"{Y}[i][j * 1] = {a['X']}[i][j * 1];")
        W.close()
        W.close()
    elif op.kind == "im2col":
        k, s, pd, H, Wd, OW = p["ksize"], p["stride"], p["pad"], p["h"], p["w"], p["ow"]
        row = f"c / {k} % {k} + h * {s} - {pd}"
        col = f"c % {k} + w * {s} - {pd}"
        W.open_for("c", p["K"])
        W.open_for("h", p["oh"])
        W.open_for("w", OW)
        W.line(f"if ({row} < 0 || {row} >= {H} || {col} < 0 || {col} >= {Wd}) {{")
        W.line(f"    {a['Y']}[c][h * {OW} + w] = 0.0;")
        W.line("} else {")
        W.line(f"    {a['Y']}[c][h * {OW} + w] = {a['X']}[c / {k * k}][({row}) * {Wd} + {col}];")
        W.line("}")
        W.close()
        W.close()
        W.close()
    elif op.kind == "gemm":
        W.open_for("i", p["M"])
        W.open_for("k", p["K"])
        W.open_for("j", p["N"])
        W.line(f"{a['C']}[i][j * 1] += {a['A']}[i][k] * {a['B']}[k][j * 1];")
        W.close()
        W.close()
        W.close()
    elif op.kind == "maxpool":
        X, Y, I = a["X"], a["Y"], a["I"]
        H, Wd, OW, st, off = p["h"], p["w"], p["ow"], p["stride"], p["off"]
        r = f"i * {st} + n - {off}"
        q = f"j * {st} + m - {off}"
        o = f"i * {OW} + j"
        W.open_for("c", p["c"])
        W.open_for("i", p["oh"])
        W.open_for("j", OW)
        W.line(f"{Y}[c][{o}] = -{FLT_MAX_LITERAL};")
        W.line(f"{I}[c][{o}] = -1;")
        W.open_for("n", p["size"])
        W.open_for("m", p["size"])
        W.line(f"if ({r} >= 0 && {r} < {H} && {q} >= 0 && {q} < {Wd}) {{")
        W.line(f"    if ({X}[c][({r}) * {Wd} + {q}] > {Y}[c][{o}]) {{")
        W.line(f"        {Y}[c][{o}] = {X}[c][({r}) * {Wd} + {q}];")
        W.line(f"        {I}[c][{o}] = c * {H * Wd} + ({r}) * {Wd} + {q};")
        W.line("    }")
        W.line("}")
        W.close()
        W.close()
        W.close()
        W.close()
        W.close()
    else:
        raise KeyError(op.kind)


# --------------------------------------------------------------------------
# seeded synthetic data (identical recipe in oracle/harness C code)
# --------------------------------------------------------------------------

_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def _fnv1a64(text: str) -> int:
    h = 0xCBF29CE484222325
    for byte in text.encode():
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def array_key(name: str, seed: int) -> int:
    return (_fnv1a64(name) ^ ((seed * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


def synth_values(name: str, seed: int, count: int, scale: float, start: int = 0) -> np.ndarray:
    """float32 values: ((splitmix64(key + i) >> 40) * 2^-24 - 0.5) * scale,
    the subtraction in double then rounded, the multiply in float."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _splitmix64(idx + np.uint64(array_key(name, seed)))
    u = (z >> np.uint64(40)).astype(np.float64) * (1.0 / 16777216.0) - 0.5
    return u.astype(np.float32) * np.float32(scale)


def array_scale(net: NetProgram, name: str) -> float:
    spec = net.arrays[name]
    if spec.role == "weight":
        return float(np.float32(math.sqrt(24.0 / spec.shape[1])))
    if spec.role == "bias":
        return 0.2
    return 2.0                                    # input images in [-1, 1)


def weight_data(net: NetProgram, name: str, seed: int) -> np.ndarray:
    spec = net.arrays[name]
    return synth_values(name, seed, spec.numel, array_scale(net, name)).reshape(spec.shape)


def input_images(net: NetProgram, seed: int, first: int, count: int) -> np.ndarray:
    """Images first..first+count-1 of the synthetic stream, (count, C, H*W)."""
    spec = net.arrays[net.input_name]
    n = spec.numel
    flat = synth_values("x", seed, n * count, array_scale(net, "x"), start=first * n)
    return flat.reshape((count,) + spec.shape)


# ------------------------------------------------- programs from their text
_PARAM = re.compile(r"^(float|int) ([A-Za-z_]\w*)((?:\[\d+\])+)$")
_CALL = re.compile(r"\b(load_input|store_output)\((\w+)\)")


class ProgramError(ValueError):
    """The source is not a Darknet-style program in the C-subset templates."""


def net_from_source(source: str, name: str = "program") -> NetProgram:
    """The NetProgram of a user-authored C-subset program,
    read off its text instead of a NETS layer list: `forward`'s parameters
    are the arrays; the loop holding `load_input(x)` / `store_output(y)` is
    the image loop; every loop directly inside it must be exactly one op as
    the templates write it (`kernel_probe.recognize`: kind, shape and
    operands are read off the headers and checked line for line).  Array
    roles follow from the ops: gemm A = weights, add_bias bias = biases,
    maxpool I = indexes, im2col Y = workspace.  Raises ProgramError."""
    from .kernel_probe import candidate_block, recognize
    from .loopnest import build_loop_tree
    from .syntax import parse
    head = re.search(r"\bint forward\(([^)]*)\)\s*\{", source)
    if head is None:
        raise ProgramError("no `int forward(...)` function")
    arrays: dict[str, ArraySpec] = {}
    for decl in (d.strip() for d in head.group(1).split(",")):
        m = _PARAM.match(decl)
        if m is None:
            raise ProgramError(f"forward parameter {decl!r} is not a float/int array")
        dims = tuple(int(v) for v in re.findall(r"\d+", m.group(3)))
        if len(dims) > 2:
            raise ProgramError(f"array {m.group(2)} has more than two dimensions")
        arrays[m.group(2)] = ArraySpec(m.group(2), m.group(1), dims, "activation")
    try:
        tree = build_loop_tree(parse(source))
    except Exception as exc:  # noqa: BLE001 -- the reference front end's errors
        raise ProgramError(f"cannot parse the program: {exc}") from exc
    tops = [n for n in tree.nodes if n.parent is None and n.function == "forward"]
    if len(tops) != 1:
        raise ProgramError("forward must hold exactly one top-level (image) loop")
    img = tops[0]
    img_text = source[img.span[0]:img.span[1]]
    calls = dict((k, v) for k, v in _CALL.findall(img_text))
    if set(calls) != {"load_input", "store_output"}:
        raise ProgramError("the image loop must call load_input(x) and store_output(y)")
    input_name, output_name = calls["load_input"], calls["store_output"]
    for v in (input_name, output_name):
        if v not in arrays or arrays[v].dtype != "float":
            raise ProgramError(f"{v} is not a float parameter of forward")
    m = re.match(r"for \((\w+) = 0; \1 < (\d+); \1\+\+\)", img_text)
    if m is None:
        raise ProgramError("the image loop header is not `for (b = 0; b < N; b++)`")
    images = int(m.group(2))
    trips, parents = [], []
    for n in tree.nodes:
        mh = re.match(r"for \((\w+) = 0; \1 < (\d+); \1\+\+\)", source[n.span[0]:n.span[1]])
        if mh is None:
            raise ProgramError(f"loop {n.loop_id} is not a counted `for` loop")
        trips.append(int(mh.group(2)))
        parents.append(n.parent)
    ops: list[OpSpec] = []
    for lid in img.children:
        node = tree.nodes[lid]
        line0 = source.rfind("\n", 0, node.span[0]) + 1          # keep the header's indent
        text = "#pragma acc kernels\n" + source[line0:node.span[1]]
        block = candidate_block(text)
        got = recognize(block) if block else None
        if got is None:
            raise ProgramError(f"loop {lid} (line {node.header_pos.line}) is not a template op")
        kind, params, ops_arrays = got
        for role, v in ops_arrays.items():
            if v not in arrays:
                raise ProgramError(f"loop {lid}: {v} is not a parameter of forward")
        ops.append(OpSpec(kind, len(ops), loop_id=lid, arrays=ops_arrays, params=params))
    for op in ops:
        a = op.arrays
        if op.kind == "gemm":
            arrays[a["A"]].role = "weight"
        elif op.kind == "add_bias":
            arrays[a["bias"]].role = "bias"
        elif op.kind == "maxpool":
            arrays[a["I"]].role = "index"
        elif op.kind == "im2col":
            arrays[a["Y"]].role = "workspace"
    arrays[input_name].role = "input"
    arrays[output_name].role = "output"
    xs = arrays[input_name].shape
    spec = NetSpec(name, xs[0] if len(xs) == 2 else 1, 0, 0, (), images)
    return NetProgram(spec, source, arrays, ops, trips, parents, img.loop_id, input_name,
                      output_name)


def write_net_files(name, outdir, images: int | None = None, auto: bool = False) -> dict:
    """Write `<name>.c`, `<name>_profile.json` and a `<name>_gpu.json`
    evaluator config -- the inputs of `tune --evaluator gpu:...`.  `name` is
    a NETS key or a NetSpec (any layer list); `auto` writes the config as
    `{"net": "auto"}` (manifest read off the source)."""
    import json
    from pathlib import Path
    net = build_net(name, images=images)
    name = net.spec.name
    out = Path(outdir)
    out.mkdir(parents=True, exist_ok=True)
    paths = {"source": out / f"{name}.c", "profile": out / f"{name}_profile.json",
             "gpu_config": out / f"{name}_gpu.json"}
    paths["source"].write_text(net.source)
    paths["profile"].write_text(json.dumps(net.profile_dict(), indent=1) + "\n")
    cfg = {"net": "auto"} if auto else {"net": name, "images": net.spec.images}
    paths["gpu_config"].write_text(json.dumps(cfg) + "\n")
    return paths


if __name__ == "__main__":
    import sys
    if len(sys.argv) < 3:
        sys.exit("usage: python -m paper_1811_03882_b200.nets <net> <outdir> [images]")
    for key, path in write_net_files(sys.argv[1], sys.argv[2],
                                     int(sys.argv[3]) if len(sys.argv) > 3 else None).items():
        print(key, path)
