"""Execute a genome's offload pattern on one B200.

`PatternExecutor(net)` owns, for one device, a pinned host buffer and a
device buffer for every array of the net's C-subset program, the seeded
weights, a pinned batch of input images and a pinned batch of output slots.
`compile(bits)` turns the genome plus its transfer plan into the flat action
list of `acct_run_schedule` (include/acct.h); `run(...)` executes it
natively and returns wall-clock seconds and the transfer/launch counters.

Semantics follow the emitted OpenACC program (reference emitter
`pkg/src/acctuner/emitter.py:41-84`, planner `transfer.py:82-158`):

* the image loop `for (b ...)` runs on the host; `load_input(x)` binds the
  host copy of `x` to image b of the pinned input batch, `store_output(y)`
  makes the host copy of `y` image b's output slot;
* every `#pragma acc data` directive executes once per arrival at its
  target loop (the count contract of `directive_exec_counts`): its
  copyin/copy variables go host->device before the loop, its copyout/copy
  variables device->host after it.  Several directives moving the same
  variable in the same direction at the same point issue one memcpy (the
  emitter merges them into one line too) but each directive is counted;
* a loop whose gene is 1 is one kernel launch on device buffers; a loop
  whose gene is 0 runs natively (acct_host_*) on host buffers, after the
  stream is drained.

B200-specific choices, none of which changes observable results:

* device arrays are pitched (rows of a multiple of 16 B, 128 B where that
  pads by <= 1/64, `_pitch`) so every row is TMA- and float4-aligned;
  transfers are pitched 2-D copies;
* with `fuse=True`, a run of consecutive offloaded ops on one conv output
  -- fill, gemm_nn, add_bias, activation -- becomes ONE gemm launch with
  beta=0 and a bias/leaky epilogue, provided no transfer of that output
  sits between them (the intermediate states are then unobservable); the
  arithmetic is the same float ops in the same order as the separate
  kernels, so outputs are bit-identical to `fuse=False`.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import kernels as K
from .errors import DeviceError, InvalidGenome
from .legality import build_genome_map, check_all_parallelizable, profile_from_dict
from .loopnest import build_loop_tree, extract_accesses
from .nets import NetProgram, input_images, weight_data
from .planner import (COPY, COPYIN, COPYOUT, TransferPlan, directive_exec_counts,
                      plan_transfers, selected_loops)
from .syntax import parse

PITCH_ALIGN = 32  # elements (128 bytes): the preferred row alignment
PITCH_MIN = 4     # elements (16 bytes): what TMA and the float4 kernels need
# 3x3/1/1 layers fused into one conv launch (im2col + gemm_nn + epilogue): at
# most CONV_MAX_C input channels and CONV_MAX_M filters.  The runtime runs
# the FP32 window kernel for M <= 16, the
# implicit-im2col tcgen05 swap tile for the other narrow layers (yolov2-tiny
# layers 2 and 4); the FP32 kernel at layer 2 (c = 16, M = 32: 199 MFMA per
# image) measured 13.7 us/img against 12.2 for im2col + the swap gemm
CONV_MAX_C = int(os.environ.get("ACCT_CONV_MAX_C", "64"))
CONV_MAX_M = int(os.environ.get("ACCT_CONV_MAX_M", "64"))
# wide layers (M a multiple of 128) on the streamed-weight tcgen05 conv:
# yolov2-tiny layer 6 (M = 128; layer 8's 26-wide rows are not TMA-describable
# as a 2-D plane, so _conv_partner's width % 4 rule keeps it unfused)
CONV_WIDE_MAX_M = int(os.environ.get("ACCT_CONV_WIDE_MAX_M", "256"))
CONV_WIDE_MAX_C = int(os.environ.get("ACCT_CONV_WIDE_MAX_C", "512"))
# wide long-K 3x3 layers (yolov2-tiny 8, 10, 12, 13; the 38x38 / 19x19
# layers of yolov2-608) as ONE launch of the CTA-pair gemm with implicit
# im2col (acct_conv3x3_gemm_tc_f32, bit-identical) -- opt-in: measured 2x
# slower than im2col + the TMA-fed gemm (yolov2-tiny L13 18.3 vs 9.0 us/img;
# four split warps cannot gather the 3 x 32 x 96 operand values per k-block
# at the MMA's pace)
IMPLICIT_GEMM = os.environ.get("ACCT_IMPLICIT_GEMM", "0") == "1"


def _pitch(cols: int) -> int:
    """Device row pitch (elements): 128-byte rows unless that pads a row by
    more than 1/64 -- the 13x13 and 19x19 planes (169 -> 172 instead of 192,
    361 -> 364 instead of 384), whose padding columns would otherwise be
    MMA columns and HBM bytes of every interleaved multi-image gemm -- then
    16-byte rows, the TMA / float4 minimum."""
    wide = -(-cols // PITCH_ALIGN) * PITCH_ALIGN
    if (wide - cols) * 64 <= cols:
        return wide
    return -(-cols // PITCH_MIN) * PITCH_MIN


def _f32_bits(v: float) -> int:
    return struct.unpack("<I", struct.pack("<f", v))[0]


@dataclass
class Schedule:
    genome: str
    actions: object                       # ctypes Action array
    n_actions: int
    plan: TransferPlan
    expected: dict                        # counters the run must reproduce
    fused_groups: list = field(default_factory=list)
    device_ops: int = 0
    host_ops: int = 0
    runs: int = 0
    graph: object = None                  # acct_graph_t* once captured (all-GPU schedules)
    graph_failed: bool = False
    batch: int = 1                        # images per launch of the image loop's body
    transfers: bool = False               # any H2D / D2H action
    slots: object = None                  # slot table of a batched schedule (None = base)


STAGE_ROW_BYTES = 4096   # the runtime stages host->device copies of shorter rows
GATHER_BYTES = int(os.environ.get("ACCT_GATHER_MB", "16")) << 20  # hoisted copyins: merged copies of <= ~16 MB
GATHER_MAX = 12          # members per merged copy (int operands of one action)


def arena_order(net: NetProgram) -> list:
    """Array order of the host arena: first touch in the op manifest (each
    op's operands in the order its kernel action lists them), arrays no op
    ever reads (maxpool indexes, the output) last -- so the copyins the
    planner hoists in front of the image loop form contiguous runs."""
    reads = set()
    for op in net.ops:
        for role, name in op.arrays.items():
            if role in ("X", "A", "B", "bias") or (role in ("C", "Y") and op.kind in
                                                     ("gemm", "add_bias", "leaky", "linear")):
                reads.add(name)
    seen, first, last = set(), [], []
    roles = ("A", "B", "C", "X", "Y", "I", "bias")
    for name in [net.input_name]:
        seen.add(name)
        first.append(name)
    for op in net.ops:
        for role in roles:
            name = op.arrays.get(role)
            if name is None or name in seen:
                continue
            seen.add(name)
            (first if name in reads else last).append(name)
    for name in net.arrays:
        if name not in seen:
            (first if name in reads else last).append(name)
    return first + last


def _carve_stages(torch, device, slots, ks, images: dict):
    """One dense device staging region PER padded short-row array (several
    images for image-major batched arrays), carved from one allocation: a
    staged copy then never waits for another array's repack to free a shared
    buffer.  Returns the backing tensor (keep it alive) or None."""
    need, offs, total = [], {}, 0
    for k in ks:
        sl = slots[k]
        if sl.ld_dev != sl.cols and sl.cols * 4 < STAGE_ROW_BYTES:
            n = sl.rows * sl.cols * images.get(k, 1)
            offs[k] = total
            total += -(-n // 64) * 64                    # 256-B aligned regions
    if not total:
        return None
    buf = torch.empty(total, dtype=torch.float32, device=device)
    for k, off in offs.items():
        slots[k].stage = buf.data_ptr() + 4 * off
    return buf


def _batched(act: tuple, nimg: int) -> tuple:
    """KERNEL action over `nimg` images per launch (int operand 13)."""
    if nimg <= 1:
        return act
    ints = list(act[2]) + [0] * (14 - len(act[2]))
    ints[13] = nimg
    return (act[0], act[1], tuple(ints)) + tuple(act[3:])


@dataclass
class RunResult:
    seconds: float
    counters: dict
    status: str = "measured"
    kernel_ms: list | None = None


class PatternExecutor:
    def __init__(self, net: NetProgram, device=0, seed: int = 1, fuse: bool = True,
                 gemm_mode: int = K.GEMM_AUTO, graphs: bool = True, first_image: int = 0,
                 batch: int | bool = True, batch_bytes: int = 48 << 30):
        import torch
        self.torch = torch
        K.lib()  # fail loudly without the kernel library
        # device=None: host-only executor (every gene 0) -- the CPU half of
        # the runner, usable without a GPU
        self.host_only = device is None
        if not self.host_only and not torch.cuda.is_available():
            raise DeviceError("PatternExecutor needs a CUDA device (sm_100a)")
        self.net = net
        self.fuse = fuse
        self.fuse_convs_single = False   # conv launches for one-image loops too (tests)
        self.gemm_mode = gemm_mode
        # image batching of the image loop (see _batch_plan): True = as many
        # images per launch as divide the step and fit `batch_bytes` of
        # private copies; an int caps the batch; False/1 = one image at a time
        self.max_batch = (1 << 30) if batch is True else max(1, int(batch or 1))
        self.batch_bytes = batch_bytes
        self.graphs = graphs and not self.host_only
        if self.host_only:
            self.device = None
        else:
            self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.program = parse(net.source)
        self.tree = build_loop_tree(self.program)
        self.accesses = extract_accesses(self.program)
        self.genome_map = build_genome_map(check_all_parallelizable(self.tree, self.accesses))
        self.profile = profile_from_dict(net.profile_dict(), net.spec.name, self.tree)
        if list(self.genome_map.loop_ids) != [op.loop_id for op in net.ops]:
            raise DeviceError("net program genes do not line up with its op manifest")
        self.images = net.spec.images

        pin = not self.host_only
        if pin:
            with torch.cuda.device(self.device):
                self.stream = torch.cuda.Stream(self.device)
        else:
            self.stream = None
        self.slot_of: dict[str, int] = {}
        self.dev: dict[str, object] = {}
        self.host: dict[str, object] = {}
        slots = (K.ArraySlot * len(net.arrays))()
        # host buffers: views into ONE pinned arena laid out in first-use order
        # (arena_order), so the hoisted copyins of a pattern are adjacent in
        # host memory and the runner can move them as a few large copies
        order = arena_order(net)
        sizes = {n: (a.shape[0] * a.shape[1] if len(a.shape) == 2 else a.shape[0])
                 for n, a in net.arrays.items()}
        self.host_offset, off = {}, 0
        for name in order:
            self.host_offset[name] = off
            off += -(-sizes[name] // 64) * 64                 # 256-B aligned
        arena = torch.zeros(max(off, 1), dtype=torch.float32, pin_memory=pin)
        self.host_arena = arena
        for k, spec in enumerate(net.arrays.values()):
            rows, cols = (spec.shape if len(spec.shape) == 2 else (1, spec.shape[0]))
            ld = _pitch(cols)
            dt = torch.float32 if spec.dtype == "float" else torch.int32
            d = None if self.host_only else torch.zeros(rows * ld, dtype=dt, device=self.device)
            o = self.host_offset[spec.name]
            h = arena[o:o + rows * cols].view(dt)
            self.dev[spec.name], self.host[spec.name] = d, h
            self.slot_of[spec.name] = k
            slots[k].host = h.data_ptr()
            slots[k].dev = None if d is None else d.data_ptr()
            slots[k].rows, slots[k].cols, slots[k].ld_dev = rows, cols, ld
        # dense staging for padded short-row arrays: their H2D is one contiguous
        # copy plus a repack kernel (short-row 2-D H2D copies run ~10x slower)
        if not self.host_only:
            self.stage = _carve_stages(torch, self.device, slots, range(len(net.arrays)), {})
        self.slots = slots
        self._pristine = [(slots[k].host, slots[k].dev) for k in range(len(net.arrays))]
        self._tables: dict[int, tuple] = {1: (slots, self._pristine)}
        self._gather_keep: list = []              # device staging of merged copyins
        self._bdev: dict[int, dict] = {}          # batch -> private device copies
        self._last_table = 1
        for spec in net.arrays.values():
            if spec.role in ("weight", "bias"):
                self.host[spec.name].copy_(torch.from_numpy(weight_data(net, spec.name, seed).ravel()))
        xs = net.arrays[net.input_name]
        self.input_batch = torch.from_numpy(
            input_images(net, seed, first_image, self.images).reshape(self.images, -1))
        self.first_image = first_image
        if pin:
            self.input_batch = self.input_batch.pin_memory()
        ys = net.arrays[net.output_name]
        self.output_batch = torch.zeros((self.images, ys.numel), dtype=torch.float32,
                                        pin_memory=pin)
        self.image_bytes = xs.numel * 4
        self.output_bytes = ys.numel * 4
        self._cache: dict[str, Schedule] = {}

    # ------------------------------------------------------------ compile
    def compile(self, genome_bits: str, resident: bool = False) -> Schedule:
        key = ("R" if resident else "E") + genome_bits
        if key in self._cache:
            return self._cache[key]
        plan = plan_transfers(self.program, self.tree, self.accesses, genome_bits, self.genome_map)
        chosen = selected_loops(genome_bits, self.genome_map)
        bp = self._batch_plan(plan, chosen)
        if resident:
            sched = self._compile_resident(genome_bits, plan, chosen, bp)
        else:
            sched = self._compile_full(genome_bits, plan, chosen, bp)
        self._cache[key] = sched
        return sched

    # ------------------------------------------------------------ batching
    def _batch_plan(self, plan: TransferPlan, chosen: set):
        """Image batching of the image loop `for (b ...)`.

        Legal when every op of the loop body is offloaded (no host loop
        inside it) and every array the body writes is private to an
        iteration: its first access in the body is a full overwrite (fill,
        im2col, copy or maxpool output; the input is rewritten by
        load_input), so no value flows from image b to image b+1.  Each
        private array then gets one device copy per image and consecutive
        iterations run as ONE launch per op over P images -- loop
        privatization + batching of an independent loop.  In-body transfers
        may only move private arrays (the input before, the output after);
        their copies are image-major so a batch moves as one block.
        Directives still count once per image, hoisted transfers before the
        loop fill image 0's copy and those after it read image P-1's copy
        (the last iteration), so the counters and every host-visible value
        equal the image-at-a-time run.  Returns None or
        (P, {array: "im" | "il"}) -- image-major / column-interleaved.
        """
        if self.host_only or self.max_batch <= 1 or self.images <= 1:
            return None
        net = self.net
        if any(op.loop_id not in chosen for op in net.ops):
            return None
        full_write = {"fill": ("Y",), "im2col": ("Y",), "copy": ("Y",), "maxpool": ("Y", "I")}
        first: dict[str, str] = {net.input_name: "w"}   # load_input(x) writes x first
        written = {net.input_name, net.output_name}
        for op in net.ops:
            outs = full_write.get(op.kind, ())
            for role, name in op.arrays.items():
                is_write = role in outs or (op.kind == "gemm" and role == "C") or \
                    (op.kind in ("add_bias", "leaky", "linear") and role == "Y")
                if is_write:
                    written.add(name)
                if name not in first:
                    first[name] = "w" if role in outs else "r"
        if any(first.get(v) != "w" for v in written):
            return None                                   # a value crosses iterations
        inside = {lid for lid in net.loop_parent} - {net.image_loop}
        moved_inside = set()
        for d in plan.directives:
            if d.target_loop in inside:
                moved_inside.update(d.vars)
        if not moved_inside <= written:
            return None
        layout = {v: ("im" if v in moved_inside or v == net.input_name else "il") for v in written}
        per_image = 0
        for v in written:
            spec = net.arrays[v]
            rows, cols = spec.shape if len(spec.shape) == 2 else (1, spec.shape[0])
            per_image += rows * _pitch(cols) * 4
        p = min(self.images, self.max_batch, max(1, self.batch_bytes // max(per_image, 1)))
        while self.images % p:
            p -= 1
        return (p, layout) if p > 1 else None

    def _batched_table(self, p: int, layout: dict):
        """Slot table for P-image batches: private arrays get P copies
        (image-major [P][rows][ld] or interleaved [rows][P*ld]); shared arrays
        (weights, biases) keep their single buffer."""
        if p in self._tables:
            return self._tables[p][0]
        torch = self.torch
        n = len(self.net.arrays)
        slots = (K.ArraySlot * n)()
        keep = []
        for k, spec in enumerate(self.net.arrays.values()):
            base = self.slots[k]
            slots[k].host, slots[k].rows, slots[k].cols = base.host, base.rows, base.cols
            slots[k].ld_dev, slots[k].dev, slots[k].img_stride = base.ld_dev, base.dev, 0
            rows, cols, ld = base.rows, base.cols, base.ld_dev
            lay = layout.get(spec.name)
            if lay is not None:
                dt = torch.float32 if spec.dtype == "float" else torch.int32
                d = torch.zeros(p * rows * ld, dtype=dt, device=self.device)
                keep.append(d)
                self._bdev.setdefault(p, {})[spec.name] = d
                slots[k].dev = d.data_ptr()
                if lay == "im":
                    slots[k].img_stride = rows * ld
                else:
                    slots[k].ld_dev, slots[k].img_stride = p * ld, ld
        images = {k: p for k, spec in enumerate(self.net.arrays.values())
                  if layout.get(spec.name) == "im"}
        stage = _carve_stages(torch, self.device, slots, range(n), images)
        if stage is not None:
            keep.append(stage)
        self._keep_alive = getattr(self, "_keep_alive", []) + keep
        pristine = [(slots[k].host, slots[k].dev) for k in range(n)]
        self._tables[p] = (slots, pristine)
        return slots

    def _compile_full(self, bits: str, plan: TransferPlan, chosen: set, bp=None) -> Schedule:
        net = self.net
        p = bp[0] if bp else 1
        acts: list[tuple] = []
        at_target: dict[int, list] = {}
        for d in plan.directives:
            at_target.setdefault(d.target_loop, []).append(d)
        in_loop = [False]

        def moves(target: int, clauses) -> list[str]:
            names = set()
            for d in at_target.get(target, ()):
                if d.clause in clauses:
                    names.update(v for v in d.vars if v in self.slot_of)
            return sorted(names)

        # transfers inside the loop move all P images of a batch; before it,
        # image 0's copy; after it, image P-1's (the last iteration's values)
        def xfer(kind, v, after=False):
            if in_loop[0]:
                return (kind, (self.slot_of[v],), (0, p, p))
            return (kind, (self.slot_of[v],), (p - 1 if after else 0, 1, 1))

        def entry(target: int):
            for d in at_target.get(target, ()):
                acts.append((K.A_DIRECTIVE, (), (len(d.vars), int(d.clause == COPY),
                                                  p if in_loop[0] else 1)))
            for v in moves(target, (COPYIN, COPY)):
                acts.append(xfer(K.A_H2D, v))

        def leave(target: int):
            for v in moves(target, (COPYOUT, COPY)):
                acts.append(xfer(K.A_D2H, v, after=not in_loop[0]))

        img = net.image_loop
        entry(img)
        begin = len(acts)
        acts.append([K.A_LOOP_BEGIN, (), (self.images // p, -1)])
        in_loop[0] = True
        x_slot, y_slot = self.slot_of[net.input_name], self.slot_of[net.output_name]
        acts.append((K.A_BIND, (x_slot,), (0, p * self.image_bytes, 0), "in"))
        # store_output(y) targets y's slot; binding y to it up front is exact
        # because every iteration overwrites y completely before reading it
        acts.append((K.A_BIND, (y_slot,), (0, p * self.output_bytes, 0), "out"))

        plan_f = self._fusion_plan(plan, chosen, p) if self.fuse else {}
        device_ops = host_ops = 0
        for n, op in enumerate(net.ops):
            role = plan_f.get(n)
            if role is None:
                entry(op.loop_id)
                on_gpu = op.loop_id in chosen
                acts.append(self._op_action(op, K.A_KERNEL if on_gpu else K.A_HOST, p))
                if on_gpu:
                    device_ops += op.kind != "linear"
                else:
                    host_ops += 1
                leave(op.loop_id)
            elif role[0] == "absorbed_before":      # fill: subsumed by beta = 0
                entry(op.loop_id)
                leave(op.loop_id)
            elif role[0] == "anchor":               # gemm (+ later bias/act)
                members = role[1]
                for m in members:
                    entry(net.ops[m].loop_id)
                acts.append(self._fused_gemm_action([net.ops[m] for m in role[2]], p, role[3],
                                                    role[4], role[5], role[6]))
                for m in members:
                    leave(net.ops[m].loop_id)
                device_ops += 1
            # role "absorbed_after": handled by its anchor
        acts.append((K.A_STORE, (y_slot,), (0, p * self.output_bytes, p * self.output_bytes), "out"))
        acts.append((K.A_LOOP_END, (), (begin,)))
        end = len(acts) - 1
        acts[begin] = (K.A_LOOP_BEGIN, (), (self.images // p, end))
        in_loop[0] = False
        leave(img)
        acts.append((K.A_SYNC, (), ()))
        expected = self._expected_counters(plan, acts)
        if bp and host_ops == 0:
            acts = self._overlap_transfers(acts, single_pass=self.images // p == 1)
        sched = self._pack(bits, acts, plan, expected)
        sched.batch = p
        if bp:
            sched.slots = self._batched_table(p, bp[1])
        sched.fused_groups = sorted((n, r[2]) for n, r in plan_f.items() if r[0] == "anchor")
        sched.device_ops, sched.host_ops = device_ops * self.images, host_ops * self.images
        return sched

    def _compile_resident(self, bits: str, plan: TransferPlan, chosen: set, bp=None) -> Schedule:
        """Kernels only, inputs already in HBM (one device batch of images):
        the `value` leg of the benchmark.  Requires every op on the GPU."""
        if len(chosen) != len(self.net.ops):
            raise InvalidGenome("resident schedules need the all-offload genome")
        if not hasattr(self, "device_batch"):
            xs = self.net.arrays[self.net.input_name]
            rows, cols = xs.shape
            ld = _pitch(cols)
            db = self.torch.zeros((self.images, rows, ld), dtype=self.torch.float32,
                                  device=self.device)
            db[:, :, :cols].copy_(self.input_batch.view(self.images, rows, cols))
            self.device_batch = db
        p = bp[0] if bp else 1
        acts: list[tuple] = []
        acts.append([K.A_LOOP_BEGIN, (), (self.images // p, -1)])
        x_slot = self.slot_of[self.net.input_name]
        rows, cols = self.net.arrays[self.net.input_name].shape
        acts.append((K.A_BIND, (x_slot,), (0, p * rows * _pitch(cols) * 4, 1), "devin"))
        plan_f = self._fusion_plan(plan, chosen, p) if self.fuse else {}
        for n, op in enumerate(self.net.ops):
            role = plan_f.get(n)
            if role is None:
                acts.append(self._op_action(op, K.A_KERNEL, p))
            elif role[0] == "anchor":
                acts.append(self._fused_gemm_action([self.net.ops[m] for m in role[2]], p,
                                                    role[3], role[4], role[5], role[6]))
        acts.append((K.A_LOOP_END, (), (0,)))
        acts[0] = (K.A_LOOP_BEGIN, (), (self.images // p, len(acts) - 1))
        acts.append((K.A_SYNC, (), ()))
        sched = self._pack(bits, acts, plan, {})
        sched.batch = p
        if bp:
            sched.slots = self._batched_table(p, bp[1])
        return sched

    @staticmethod
    def _written_slots(act) -> tuple:
        """Array slots a KERNEL action writes."""
        kind, slots = act[2][0], act[1]
        if kind in (K.K_FILL, K.K_ADD_BIAS, K.K_LEAKY, K.K_LINEAR):
            return (slots[0],)
        if kind in (K.K_COPY, K.K_IM2COL):
            return (slots[1],)
        if kind == K.K_GEMM:
            return (slots[2],)
        if kind == K.K_MAXPOOL:
            return (slots[1], slots[2])
        if kind == K.K_CONV:
            return (slots[1], slots[3]) + tuple(v for v in act[2][9:11] if v >= 0)
        return ()

    def _overlap_transfers(self, acts: list, single_pass: bool) -> list:
        """Reorder the transfers of an all-device schedule for overlap; the
        set of transfers, their directions and counts are unchanged.

        * hoisted copyins in front of the image loop (all at one program
          point, so their mutual order is free) go out in order of first use
          in the loop body -- the runner streams them on a side stream and
          each kernel waits only for its own operands;
        * when the loop body runs once (one batch = every image), a hoisted
          copyout after the loop moves up to just after the last kernel that
          writes the array (no later action changes it), flagged early: the
          runner issues it on a device->host side stream while the remaining
          layers compute.
        """
        begin = next(i for i, a in enumerate(acts) if a[0] == K.A_LOOP_BEGIN)
        end = next(i for i, a in enumerate(acts) if a[0] == K.A_LOOP_END)
        pre, body, post = list(acts[:begin]), list(acts[begin + 1:end]), list(acts[end + 1:])
        first_use: dict[int, int] = {}
        for i, a in enumerate(body):
            slots = tuple(a[1])
            if a[0] == K.A_KERNEL and a[2][0] == K.K_CONV:
                slots += (a[2][7],)                    # the conv's bias slot
            for slot in slots:
                if slot is not None and slot >= 0:
                    first_use.setdefault(slot, i)
        h2d = [a for a in pre if a[0] == K.A_H2D]
        rest = [a for a in pre if a[0] != K.A_H2D]
        h2d.sort(key=lambda a: first_use.get(a[1][0], len(body)))
        pre = rest + self._gather(h2d)
        if single_pass:
            last_write: dict[int, int] = {}
            for i, a in enumerate(body):
                if a[0] == K.A_KERNEL:
                    for slot in self._written_slots(a):
                        last_write[slot] = i
            inserts: dict[int, list] = {}
            kept = []
            for a in post:
                if a[0] == K.A_D2H and a[1][0] in last_write:
                    ints = tuple(a[2]) + (0,) * (4 - len(a[2]))
                    early = (a[0], a[1], ints[:3] + (1,) + ints[4:])
                    inserts.setdefault(last_write[a[1][0]], []).append(early)
                else:
                    kept.append(a)
            new_body = []
            for i, a in enumerate(body):
                new_body.append(a)
                new_body.extend(inserts.get(i, ()))
            body, post = new_body, kept
        trip = acts[begin][2][0]
        out = pre + [None] + body + [None] + post
        b, e = len(pre), len(pre) + 1 + len(body)
        out[b] = (K.A_LOOP_BEGIN, (), (trip, e))
        out[e] = (K.A_LOOP_END, (), (b,))
        return out

    def _gather(self, h2d: list) -> list:
        """Merge runs of whole-array copyins whose host buffers are adjacent in
        the pinned arena into A_H2D_GATHER actions (one copy of up to
        GATHER_BYTES + one scatter kernel each): many small host->device
        copies interleaved with device->host ones run far below the PCIe
        duplex rate (57 copies: 4.6 ms vs 3.7 ms for the same bytes as 8,
        tools/duplex_probe.py).  Order is kept; counts are unchanged."""
        if self.host_only or not h2d:
            return h2d
        names = list(self.net.arrays)
        spans = []
        for a in h2d:
            if len(a[2]) > 1 and (a[2][0] != 0 or a[2][1] > 1):
                spans.append(None)                      # not a whole-array copy
                continue
            spec = self.net.arrays[names[a[1][0]]]
            off = self.host_offset[spec.name] * 4
            spans.append((off, off + spec.numel * 4))
        # arena order within the run keeps neighbours adjacent
        idx = sorted(range(len(h2d)), key=lambda i: spans[i][0] if spans[i] else -1)
        out, group = [], []

        def flush():
            if not group:
                return
            if len(group) == 1:
                out.append(h2d[group[0]])
            else:
                lo = spans[group[0]][0]
                hi = spans[group[-1]][1]
                stage = self.torch.empty(-(-(hi - lo) // 4), dtype=self.torch.float32,
                                         device=self.device)
                self._gather_keep.append(stage)
                ints = [len(group)] + [h2d[i][1][0] for i in group]
                ints += [0] * (13 - len(ints)) + [stage.data_ptr()]
                out.append((K.A_H2D_GATHER, (), tuple(ints), self.host_arena.data_ptr() + lo))
            group.clear()

        for i in idx:
            if spans[i] is None:
                flush()
                out.append(h2d[i])
                continue
            if group:
                last = spans[group[-1]]
                size = spans[i][1] - spans[group[0]][0]
                if (spans[i][0] - last[1] > 256 or size > GATHER_BYTES or len(group) >= GATHER_MAX):
                    flush()
            group.append(i)
        flush()
        return out

    def _fusion_plan(self, plan: TransferPlan, chosen: set, nimg: int = 1) -> dict:
        """Per conv layer, fuse offloaded fill -> gemm -> add_bias -> activation
        of one output array into a single gemm launch.

        Returns {op index: role}: ("absorbed_before",) for a fused fill,
        ("anchor", [ops whose directives execute around the launch],
        [fused op indices], im2col index or None) for the gemm,
        ("absorbed_after",) for a fused bias/activation, ("absorbed_conv",)
        for an im2col folded into the launch (see _conv_partner).  A member joins only if it is offloaded and no
        directive moves the output array at any loop boundary strictly
        inside the fused span (so its intermediate values are unobservable);
        ops in between that do not touch the output (im2col) run unchanged.
        """
        moved: dict[int, set] = {}
        for d in plan.directives:
            moved.setdefault(d.target_loop, set()).update(d.vars)
        ops = self.net.ops
        on = [op.loop_id in chosen for op in ops]
        roles: dict[int, tuple] = {}
        for g, op in enumerate(ops):
            if op.kind != "gemm" or not on[g]:
                continue
            out = op.arrays["C"]
            touches = lambda i: out in ops[i].arrays.values()  # noqa: E731
            blocked = lambda i: out in moved.get(ops[i].loop_id, set())  # noqa: E731
            # backwards: the layer's fill, across ops that never touch `out`
            fill = None
            i = g - 1
            while i >= 0 and not touches(i):
                i -= 1
            if i >= 0 and ops[i].kind == "fill" and ops[i].arrays["Y"] == out and on[i] \
                    and not any(blocked(j) for j in range(i, g + 1)):
                fill = i
            after = []
            j = g + 1
            for kind in ("add_bias", "act"):
                if j < len(ops) and on[j] and ops[j].arrays.get("Y") == out and \
                        (ops[j].kind == kind or (kind == "act" and ops[j].kind in ("leaky", "linear"))):
                    if blocked(j - 1) or blocked(j):
                        break
                    # the previous member's exit must not move `out` either
                    after.append(j)
                    j += 1
                else:
                    break
            if after and blocked(g):
                after = []
            fused = ([fill] if fill is not None else []) + [g] + after
            if len(fused) < 2:
                continue
            # conv launches (im2col joined to the gemm) only for batched
            # loops: one image leaves their pipelines a handful of units per
            # SM, and im2col + the gemm (split-K) measured faster -- the
            # image-at-a-time yolov2-tiny step 3.48 -> 2.96 ms per 16 images
            conv = self._conv_partner(g, on, moved) \
                if nimg > 1 or self.fuse_convs_single else None
            # the implicit-im2col pair gemm fuses no maxpool (it stays a launch)
            pool = self._pool_partner(g, after, on, blocked) \
                if conv is not None and not self._implicit_conv(conv) else None
            if fill is not None:
                roles[fill] = ("absorbed_before",)
            if conv is not None:
                roles[conv] = ("absorbed_conv",)
            tail = after + ([pool] if pool is not None else [])
            roles[g] = ("anchor", ([conv] if conv is not None else []) + [g] + tail, fused, conv,
                        conv is not None and self._col_dead(conv, g, moved), pool,
                        pool is not None and self._out_dead(g, fill, after, pool, moved))
            for j in tail:
                roles[j] = ("absorbed_after",)
        return roles

    def _pool_partner(self, g: int, after: list, on: list, blocked):
        """The 2x2/2 maxpool reading the output of a fused conv launch, when it
        can join the launch (acct_conv3x3_*_f32 with pool): it directly
        follows the launch's last member, is offloaded, pools the conv output
        over even planes with darknet's offset 0, and no directive at the last
        member's or the maxpool's loop boundary moves the output (a copyin
        there would change what the maxpool reads)."""
        ops = self.net.ops
        last = after[-1] if after else g
        j = last + 1
        if j >= len(ops) or not on[j] or ops[j].kind != "maxpool":
            return None
        op, q = ops[j], ops[j].params
        if op.arrays["X"] != ops[g].arrays["C"]:
            return None
        if (q["size"], q["stride"], q["off"]) != (2, 2, 0) or q["h"] % 2 or q["w"] % 2:
            return None
        if blocked(last) or blocked(j):
            return None
        return j

    def _out_dead(self, g: int, fill, after: list, pool: int, moved: dict) -> bool:
        """True when, in an image-batched run, only the LAST image's copy of a
        pooled conv output is observable: the output is touched only by the
        layer's fill, gemm, bias / activation and the fused maxpool, and no
        directive inside the image loop moves it (so the fused launch stores
        it for the batch's last image only)."""
        net = self.net
        out = net.ops[g].arrays["C"]
        own = {g, pool, *after} | ({fill} if fill is not None else set())
        if any(out in op.arrays.values() for k, op in enumerate(net.ops) if k not in own):
            return False
        return not any(out in vs for lid, vs in moved.items() if lid != net.image_loop)

    def _col_dead(self, im: int, g: int, moved: dict) -> bool:
        """True when, in an image-batched run, only the LAST image's copy of
        the fused conv's col array is observable: no directive inside the
        image loop moves col (hoisted copyouts after the loop read image
        P-1's copy; hoisted copyins land in image 0's copy and are
        overwritten by the im2col) and no op but the im2col and its gemm
        touches it.  The other images' col stores are then dead (the gemm
        reads the fused launch's registers, not col) and the kernel skips
        them -- 18.7 of the 32 MB the 416x416 first layer moves per image."""
        net = self.net
        col = net.ops[im].arrays["Y"]
        if any(col in op.arrays.values() for k, op in enumerate(net.ops) if k not in (im, g)):
            return False
        return not any(col in vs for lid, vs in moved.items() if lid != net.image_loop)

    def _implicit_conv(self, im: int) -> bool:
        """True when the fused conv of im2col op `im` runs on the CTA-pair
        gemm with implicit im2col (the runtime's choice, acct_runtime.cu
        ACCT_K_CONV): neither the narrow nor the wide conv kernel takes it."""
        p = self.net.ops[im].params
        M = self.net.ops[im + 1].params["M"]
        narrow = p["c"] <= CONV_MAX_C and M <= CONV_MAX_M
        wide = M % 128 == 0 and M <= CONV_WIDE_MAX_M and p["c"] <= CONV_WIDE_MAX_C \
            and p["w"] % 4 == 0
        return not (narrow or wide)

    def _conv_partner(self, g: int, on: list, moved: dict):
        """The im2col feeding gemm `g`, when the two can run as one fused
        conv launch (acct_conv3x3_im2col_gemm_f32): the im2col is offloaded
        and directly precedes the gemm, is 3x3/1/1 over <= CONV_MAX_C
        channels with M <= CONV_MAX_M filters (the narrow layers, whose gemm
        would stream col from HBM), and no directive between
        the two moves the input, col or output -- so moving the col write to
        the gemm's launch point is unobservable."""
        ops = self.net.ops
        if g == 0:
            return None
        op, im = ops[g], ops[g - 1]
        p = im.params
        if im.kind != "im2col" or not on[g - 1] or im.arrays["Y"] != op.arrays["B"]:
            return None
        if (p["ksize"], p["stride"], p["pad"]) != (3, 1, 1):
            return None
        M = op.params["M"]
        narrow = p["c"] <= CONV_MAX_C and M <= CONV_MAX_M
        wide = M % 128 == 0 and M <= CONV_WIDE_MAX_M and p["c"] <= CONV_WIDE_MAX_C
        # the CTA-pair gemm gathering its B operand from the input planes
        # (acct_conv3x3_gemm_tc_f32): any plane width, M >= 256, K > 768
        implicit = IMPLICIT_GEMM and M >= 256 and 9 * p["c"] > 768
        if not (narrow or wide or implicit):
            return None
        if p["w"] % 4 and not implicit:
            return None
        # the launch runs after both entries and before both exits: a copyout
        # at the im2col's exit must not see C early, a copyin at the gemm's
        # entry must not change what the im2col read or wrote
        if {im.arrays["Y"], op.arrays["C"]} & moved.get(im.loop_id, set()):
            return None
        if {im.arrays["X"], im.arrays["Y"]} & moved.get(op.loop_id, set()):
            return None
        return g - 1

    def _fused_gemm_action(self, members, nimg: int = 1, conv=None, col_dead=False, pool=None,
                           out_dead=False):
        kinds = [m.kind for m in members]
        g = next(m for m in members if m.kind == "gemm")
        p, a = g.params, g.arrays
        bias_slot = -1
        act = K.ACT_NONE
        for m in members:
            if m.kind == "add_bias":
                bias_slot = self.slot_of[m.arrays["bias"]]
            elif m.kind == "leaky":
                act = K.ACT_LEAKY
            elif m.kind == "linear":
                act = K.ACT_LINEAR
        beta_one = 0 if "fill" in kinds else 1
        if conv is not None:
            im = self.net.ops[conv]
            q = im.params
            return _batched((K.A_KERNEL, (self.slot_of[im.arrays["X"]], self.slot_of[a["B"]],
                                          self.slot_of[a["A"]], self.slot_of[a["C"]]),
                             (K.K_CONV, q["c"], q["h"], q["w"], p["M"], beta_one, act,
                              bias_slot, int(col_dead and nimg > 1),
                              self.slot_of[self.net.ops[pool].arrays["Y"]] if pool is not None else -1,
                              self.slot_of[self.net.ops[pool].arrays["I"]] if pool is not None else -1,
                              int(out_dead and nimg > 1))), nimg)
        return _batched((K.A_KERNEL, (self.slot_of[a["A"]], self.slot_of[a["B"]],
                                      self.slot_of[a["C"]], bias_slot),
                         (K.K_GEMM, p["M"], p["N"], p["K"], beta_one, act)), nimg)

    def _op_action(self, op, where: int, nimg: int = 1):
        return _batched(self._op_action1(op, where), nimg)

    def _op_action1(self, op, where: int):
        s, p, a = self.slot_of, op.params, op.arrays
        kind = op.kind
        if kind == "fill":
            return (where, (s[a["Y"]],), (K.K_FILL, p["M"], p["N"], _f32_bits(0.0)))
        if kind == "copy":
            return (where, (s[a["X"]], s[a["Y"]]), (K.K_COPY, p["M"], p["N"]))
        if kind == "im2col":
            return (where, (s[a["X"]], s[a["Y"]]),
                    (K.K_IM2COL, p["c"], p["h"], p["w"], p["ksize"], p["stride"], p["pad"]))
        if kind == "gemm":
            return (where, (s[a["A"]], s[a["B"]], s[a["C"]], -1),
                    (K.K_GEMM, p["M"], p["N"], p["K"], 1, K.ACT_NONE))
        if kind == "add_bias":
            return (where, (s[a["Y"]], s[a["bias"]]), (K.K_ADD_BIAS, p["M"], p["N"]))
        if kind in ("leaky", "linear"):
            return (where, (s[a["Y"]],),
                    (K.K_LEAKY if kind == "leaky" else K.K_LINEAR, p["M"], p["N"]))
        if kind == "maxpool":
            return (where, (s[a["X"]], s[a["Y"]], s[a["I"]]),
                    (K.K_MAXPOOL, p["c"], p["h"], p["w"], p["size"], p["stride"], p["off"],
                     p["oh"], p["ow"]))
        raise KeyError(kind)

    def _expected_counters(self, plan: TransferPlan, acts) -> dict:
        counts = directive_exec_counts(plan, self.tree, self.profile)
        execs = sum(counts.values())
        var_xfers = sum(n * len(d.vars) * (2 if d.clause == COPY else 1) for d, n in counts.items())
        # memcpy calls: actions inside the image loop run `images` times
        inside = False
        h2d = d2h = h2d_b = d2h_b = 0
        for act in acts:
            kind = act[0]
            if kind == K.A_LOOP_BEGIN:
                inside = True
            elif kind == K.A_LOOP_END:
                inside = False
            elif kind in (K.A_H2D, K.A_D2H):
                spec = list(self.net.arrays.values())[act[1][0]]
                ints = act[2]
                per = max(ints[2], 1) if len(ints) > 2 else 1   # transfers the action stands for
                reps = (self.images // per) * per if inside else 1
                if kind == K.A_H2D:
                    h2d += reps
                    h2d_b += reps * spec.nbytes
                else:
                    d2h += reps
                    d2h_b += reps * spec.nbytes
        return {"directive_execs": execs, "var_transfers": var_xfers, "h2d_calls": h2d,
                "d2h_calls": d2h, "h2d_bytes": h2d_b, "d2h_bytes": d2h_b}

    def _pack(self, bits, acts, plan, expected) -> Schedule:
        arr = (K.Action * len(acts))()
        for n, act in enumerate(acts):
            kind, slots, ints = act[0], act[1], act[2]
            arr[n].kind = kind
            for j in range(4):
                arr[n].a[j] = slots[j] if j < len(slots) else -1
            for j, v in enumerate(ints):
                arr[n].i[j] = int(v)
            if len(act) > 3 and isinstance(act[3], int):
                arr[n].base = act[3]                      # raw host pointer (gather)
            elif len(act) > 3:
                arr[n].base = {"in": self.input_batch.data_ptr(),
                               "out": self.output_batch.data_ptr(),
                               "devin": getattr(self, "device_batch", None).data_ptr()
                               if act[3] == "devin" else 0}[act[3]]
        sched = Schedule(bits, arr, len(acts), plan, expected)
        sched.transfers = any(a[0] in (K.A_H2D, K.A_D2H) for a in acts)
        return sched

    # ------------------------------------------------------------ run
    def _table(self, schedule: Schedule):
        p = schedule.batch if schedule.slots is not None else 1
        return self._tables[p][0], p

    def _restore_slots(self, p: int = None):
        for q in ([p] if p is not None else list(self._tables)):
            slots, pristine = self._tables[q]
            for k, (h, d) in enumerate(pristine):
                slots[k].host, slots[k].dev = h, d

    def run(self, schedule: Schedule | str, timeout_s: float = 0.0, resident: bool = False,
            profile: bool = False) -> RunResult:
        """Execute a compiled pattern.  With `profile=True` the result's
        `kernel_ms` holds the summed device milliseconds of every kernel
        action (CUDA events on the launch stream)."""
        if isinstance(schedule, str):
            schedule = self.compile(schedule, resident=resident)
        if self.host_only and "1" in schedule.genome:
            raise DeviceError("host-only executor can only run the all-zero genome")
        lib = K.lib()
        slots, p = self._table(schedule)
        self._last_table = p
        self._restore_slots(p)
        K.reset_counters()
        kernel_ms = (C.c_float * schedule.n_actions)() if profile else None

        def go(stream):
            t0 = time.perf_counter()
            if profile:
                rc = lib.acct_run_schedule_profiled(
                    slots, len(self.net.arrays), schedule.actions, schedule.n_actions,
                    self.gemm_mode, float(timeout_s), C.c_void_p(stream), kernel_ms)
            else:
                rc = lib.acct_run_schedule(slots, len(self.net.arrays), schedule.actions,
                                           schedule.n_actions, self.gemm_mode, float(timeout_s),
                                           C.c_void_p(stream))
            return rc, time.perf_counter() - t0

        if self.host_only:
            rc, seconds = go(0)
        else:
            with self.torch.cuda.device(self.device):
                # graphs pay off for launch-bound schedules (image at a time, or
                # batched without transfers); a batched schedule with transfers
                # is PCIe-bound and its side-stream copies ran ~6% slower as
                # graph memcpy nodes (tools/e2e_probe.py)
                launch_bound = schedule.batch == 1 or not schedule.transfers
                if (self.graphs and launch_bound and not profile and schedule.host_ops == 0
                        and schedule.runs >= 1 and not schedule.graph_failed):
                    return self._replay(schedule, timeout_s)
                rc, seconds = go(self.stream.cuda_stream)
        self._restore_slots(p)
        schedule.runs += 1
        if rc == K.ETIMEOUT:
            return RunResult(seconds, K.counters(), "timeout")
        K.check(rc, f"acct_run_schedule({schedule.genome})")
        res = RunResult(seconds, K.counters())
        if profile:
            res.kernel_ms = list(kernel_ms)
        return res

    def _replay(self, schedule: Schedule, timeout_s: float) -> RunResult:
        """All-GPU schedules: capture the whole action list into one CUDA
        graph on the second run (the first warmed lazily allocated scratch),
        then every run is a single graph launch.  Counters are re-applied by
        the library per replay."""
        lib = K.lib()
        stream = C.c_void_p(self.stream.cuda_stream)
        slots, p = self._table(schedule)
        if schedule.graph is None:
            handle = C.c_void_p()
            rc = lib.acct_schedule_capture(slots, len(self.net.arrays), schedule.actions,
                                           schedule.n_actions, self.gemm_mode, stream,
                                           C.byref(handle))
            self._restore_slots(p)
            if rc != 0 or not handle.value:
                schedule.graph_failed = True
                K.lib().acct_counters_reset()
                return self.run(schedule, timeout_s)
            schedule.graph = handle
            import weakref
            weakref.finalize(schedule, lib.acct_graph_destroy, handle)
        K.reset_counters()
        t0 = time.perf_counter()
        rc = lib.acct_graph_replay(schedule.graph, stream, 1)
        seconds = time.perf_counter() - t0
        K.check(rc, f"acct_graph_replay({schedule.genome})")
        schedule.runs += 1
        status = "timeout" if (timeout_s > 0 and seconds > timeout_s) else "measured"
        return RunResult(seconds, K.counters(), status)

    def action_op(self, schedule: Schedule, k: int) -> dict:
        """Describe KERNEL action k: op kind, shape ints and the algorithmic
        bytes / flops one execution of it performs."""
        a = schedule.actions[k]
        kind = int(a.i[0])
        ops = [op for op in self.net.ops]
        name = {v: n for n, v in K.OP_KIND.items()}[kind]
        i = [int(a.i[j]) for j in range(14)]
        slots = list(self.net.arrays.values())
        nimg = max(i[13], 1)                       # images per launch
        execs = self.images // nimg                # launches per run (body of the image loop)
        if kind == K.K_GEMM:
            M, N, Kd = i[1], i[2], i[3]
            c_bytes = (4 if i[4] else 0) + 4        # read C only when beta = 1
            bias = 4 * M if a.a[3] >= 0 else 0
            # the weights are read once per launch, whatever the batch
            byts = 4 * M * Kd + nimg * (4 * Kd * N + c_bytes * M * N) + bias
            op = next(o for o in ops if o.kind == "gemm" and o.arrays["C"] == slots[a.a[2]].name)
            # the launch's column count: images interleaved at the array pitch
            n_launch = (nimg - 1) * _pitch(N) + N if nimg > 1 else N
            return {"kind": "gemm", "layer": op.layer, "M": M, "N": N, "K": Kd, "images": nimg,
                    "N_launch": n_launch,
                    "executions": execs, "flops": 2 * M * N * Kd * nimg, "bytes": byts,
                    "fused": a.a[3] >= 0 or i[4] == 0}
        if kind == K.K_CONV:
            c, h, w, M = i[1], i[2], i[3], i[4]
            N, Kd = h * w, 9 * c
            op = next(o for o in ops if o.kind == "gemm" and o.arrays["C"] == slots[a.a[3]].name)
            # input image in, col + C out (C also in when beta = 1), weights once;
            # col of the last image only when the others are dead (i[8]), C
            # likewise when a fused maxpool consumes it (i[11]); pool + idx out
            col_imgs = 1 if i[8] else nimg
            c_imgs = 1 if i[11] else nimg
            pooled = i[9] >= 0
            byts = 4 * M * Kd + nimg * 4 * (c * N + (M * N if i[5] else 0)) + \
                c_imgs * 4 * M * N + col_imgs * 4 * Kd * N + \
                (nimg * 8 * M * (N // 4) if pooled else 0)
            byts += 4 * M if i[7] >= 0 else 0
            # the runtime's engine choice (acct_runtime.cu, ACCT_K_CONV)
            fp32 = self.gemm_mode == K.GEMM_SIMT or (self.gemm_mode == K.GEMM_AUTO and (
                M <= 16 or (M <= 32 and c <= 4 and i[9] >= 0)))
            implicit = not fp32 and M >= 256 and Kd > 768 and (M > 256 or w % 4 != 0)
            engine = "fp32-fma" if fp32 else ("tcgen05 pair, implicit im2col" if implicit
                                              else "tcgen05")
            return {"kind": "conv", "engine": engine,
                    "layer": op.layer, "M": M, "N": N, "K": Kd, "images": nimg,
                    "N_launch": (nimg - 1) * _pitch(N) + N if implicit and nimg > 1 else N,
                    "executions": execs, "flops": 2 * M * N * Kd * nimg,
                    "bytes": byts, "fused": True}
        target = slots[a.a[0]].name
        op = next(o for o in ops if o.kind == name and target in o.arrays.values())
        return {"kind": name, "layer": op.layer, "images": nimg, "executions": execs, "flops": 0,
                "bytes": op.algorithmic_bytes() * nimg, "fused": False}

    def outputs(self) -> np.ndarray:
        """(images, C, H*W) copy of the output slots after a run."""
        spec = self.net.arrays[self.net.output_name]
        return self.output_batch.numpy().reshape((self.images,) + spec.shape).copy()

    def device_array(self, name: str) -> np.ndarray:
        """Logical (unpitched) contents of a device array."""
        spec = self.net.arrays[name]
        rows, cols = spec.shape if len(spec.shape) == 2 else (1, spec.shape[0])
        p = self._last_table
        priv = self._bdev.get(p, {}).get(name)
        if priv is None:
            d = self.dev[name].view(rows, _pitch(cols))[:, :cols]
            return d.cpu().numpy().reshape(spec.shape)
        # batched schedule: the last image's private copy (what the
        # image-at-a-time loop leaves in the array)
        slot = self._tables[p][0][self.slot_of[name]]
        view = priv[(p - 1) * slot.img_stride:].as_strided((rows, cols), (slot.ld_dev, 1))
        return view.cpu().numpy().reshape(spec.shape)

    def device_outputs(self) -> np.ndarray:
        """(images, C, H*W) of the output array's private device copies after
        a batched run whose one batch is every image (the resident leg of the
        benchmark: no output slots are written there)."""
        p = self._last_table
        name = self.net.output_name
        priv = self._bdev.get(p, {}).get(name)
        if priv is None or p != self.images:
            raise DeviceError("device_outputs: needs a batched run over all images at once")
        spec = self.net.arrays[name]
        rows, cols = spec.shape
        slot = self._tables[p][0][self.slot_of[name]]
        view = priv.as_strided((p, rows, cols), (slot.img_stride, slot.ld_dev, 1))
        return view.cpu().numpy().copy()

    def host_array(self, name: str) -> np.ndarray:
        spec = self.net.arrays[name]
        return self.host[name].numpy().reshape(spec.shape).copy()
