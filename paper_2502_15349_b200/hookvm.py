"""Whole-tensor elementwise hooks on the GPU (``af_hook_eval``, csrc/hook_vm.cu).

The template kernels fuse the score / mask / online hooks into their register epilogues
(``plan.py``).  The remaining elementwise hooks act on a whole tensor and are evaluated here:

* ``output_mod`` on either template (the reference applies it to the full output,
  engine.py:502-504, 548-550, 613-615);
* ``q_mod`` / ``k_mod`` / ``v_mod`` that are neither a compile-time scalar nor one of
  ``af_feature_map``'s fixed forms — e.g. ones reading a per-head or per-step extra, or the
  position grid ``qidx`` (engine.py:511-522, 445-452).

``compile_hook`` turns a hook AST (``hooklang``) into the postfix program of
``af_hook_program``: names resolve to tensor operands (the hook's input and the spec's extras),
dims constants fold, ``qidx``/``kidx`` become the element's sequence coordinate.  ``run_hook``
launches it for one [B, H, S, D] grid and can return, in the same pass, ``seed * d hook / d x``
for one operand x — the hook's VJP (reference adjoint rules, graph.py:481-569).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import hooklang as H
from . import runtime as rt
from .errors import InputError, ShapeError, UnsupportedError

OP_OPERAND, OP_CONST, OP_INDEX = 1, 2, 3
_BIN = {"+": 11, "-": 12, "*": 13, "/": 14}
_UN = {"exp": 20, "exp2": 21, "log": 22, "abs": 23, "tanh": 24, "sigmoid": 25, "relu": 26,
       "sqrt": 27}
_FN2 = {"max": 30, "min": 31}
_CMP = {"<": 40, "<=": 41, ">": 42, ">=": 43, "==": 44, "!=": 45}
OP_NEG, OP_CLAMP, OP_WHERE = 10, 32, 33
MAX_OPS, MAX_CONSTS, MAX_OPERANDS, MAX_STACK = 128, 32, 8, 16


class HookProgram(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("ops", C.c_int32 * MAX_OPS), ("n_consts", C.c_int32),
                ("consts", C.c_float * MAX_CONSTS)]


class HookOperand(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("dtype", C.c_int32), ("stride", C.c_int64 * 4)]


@dataclass(frozen=True)
class CompiledHook:
    source: str
    ops: tuple[int, ...]
    consts: tuple[float, ...]
    operands: tuple[str, ...]      # operand index -> tensor name

    def uses(self, name: str) -> bool:
        return name in self.operands


def compile_hook(fn, inputs, consts: dict, *, index_names=("qidx",)) -> CompiledHook:
    """Compile a ``ModificationFn`` (or bare AST) over tensor names ``inputs`` (in operand order;
    only the ones the expression reads become operands).  ``index_names`` map to an element
    coordinate: a sequence of names (all the row axis, 2) or a {name: axis} dict (score grids:
    qidx -> 2, kidx -> 3).  Raises ``UnsupportedError`` for reductions or programs beyond the
    kernel's limits."""
    axes = dict(index_names) if isinstance(index_names, dict) else {n: 2 for n in index_names}
    expr = H.fold(getattr(fn, "expr", fn), consts)
    source = getattr(fn, "source", H.to_source(expr))
    ops: list[int] = []
    cvals: list[float] = []
    used: list[str] = []
    depth = [0, 0]

    def push(n=1):
        depth[0] += n
        depth[1] = max(depth[1], depth[0])

    def emit(e):
        if isinstance(e, H.Num):
            if e.value not in cvals:
                cvals.append(e.value)
            ops.extend((OP_CONST, cvals.index(e.value)))
            push()
        elif isinstance(e, H.Name):
            if e.name in axes:
                ops.extend((OP_INDEX, axes[e.name]))
            elif e.name in inputs:
                if e.name not in used:
                    used.append(e.name)
                ops.extend((OP_OPERAND, used.index(e.name)))
            else:
                raise UnsupportedError("hook reads a name that is not an input, an extra or a "
                                       "dims constant", name=e.name, source=source)
            push()
        elif isinstance(e, H.Neg):
            emit(e.operand)
            ops.append(OP_NEG)
        elif isinstance(e, (H.BinOp, H.Cmp)):
            emit(e.lhs)
            emit(e.rhs)
            ops.append((_BIN if isinstance(e, H.BinOp) else _CMP)[e.op])
            depth[0] -= 1
        elif isinstance(e, H.Fn):
            if e.func in H.REDUCTIONS:
                raise UnsupportedError("row reductions are not elementwise hooks", source=source)
            for a in e.args:
                emit(a)
            if e.func in _UN:
                ops.append(_UN[e.func])
            elif e.func in _FN2:
                ops.append(_FN2[e.func])
                depth[0] -= 1
            elif e.func == "clamp":
                ops.append(OP_CLAMP)
                depth[0] -= 2
            elif e.func == "where":
                ops.append(OP_WHERE)
                depth[0] -= 2
            else:
                raise UnsupportedError("unknown hook function", func=e.func, source=source)
        else:
            raise InputError("not a hook expression", form=type(e).__name__)

    emit(expr)
    if len(ops) > MAX_OPS or len(cvals) > MAX_CONSTS or len(used) > MAX_OPERANDS \
            or depth[1] > MAX_STACK:
        raise UnsupportedError("hook program exceeds the kernel's limits", source=source,
                               ops=len(ops), consts=len(cvals), operands=len(used),
                               stack=depth[1])
    return CompiledHook(source, tuple(ops), tuple(cvals), tuple(used))


def _operand(t: torch.Tensor, shape: tuple, name: str) -> tuple[HookOperand, torch.Tensor]:
    if not t.is_cuda:
        raise InputError("hook operands must be CUDA tensors", name=name)
    if t.dtype not in (torch.bfloat16, torch.float32):
        t = t.to(torch.float32)
    if t.dim() != 4:
        raise ShapeError("hook operands are rank 4", name=name, got=tuple(t.shape))
    st = []
    for i in range(4):
        if t.shape[i] == shape[i]:
            st.append(int(t.stride(i)) if shape[i] > 1 else 0)
        elif t.shape[i] == 1:
            st.append(0)
        else:
            raise ShapeError("hook operand does not broadcast to the hook grid", name=name,
                             got=tuple(t.shape), grid=tuple(shape))
    op = HookOperand(t.data_ptr(), rt.AF_DTYPE_BF16 if t.dtype == torch.bfloat16
                     else rt.AF_DTYPE_F32, (C.c_int64 * 4)(*st))
    return op, t


def run_hook(hook: CompiledHook, shape, tensors: dict, *, out_dtype=torch.bfloat16,
             value: bool = True, wrt: str | None = None, seed: torch.Tensor | None = None,
             deriv_dtype=torch.float32):
    """Evaluate ``hook`` over the [B, H, S, D] grid ``shape``: returns (value or None,
    seed * d hook / d wrt or None).  Freshly allocated contiguous outputs."""
    shape = tuple(int(x) for x in shape)
    keep = []
    ops = (HookOperand * MAX_OPERANDS)()
    dev = None
    for i, name in enumerate(hook.operands):
        if name not in tensors:
            raise InputError("missing hook operand", name=name, hook=hook.source)
        ops[i], t = _operand(tensors[name], shape, name)
        keep.append(t)
        dev = t.device
    if dev is None:
        dev = next(iter(tensors.values())).device
    prog = HookProgram()
    prog.n_ops = len(hook.ops)
    for i, x in enumerate(hook.ops):
        prog.ops[i] = x
    prog.n_consts = len(hook.consts)
    for i, x in enumerate(hook.consts):
        prog.consts[i] = x
    out = torch.empty(shape, device=dev, dtype=out_dtype) if value else None
    der = None
    w = -1
    seed_op = None
    if wrt is not None:
        if wrt not in hook.operands:  # the hook does not read it: derivative 0
            der = torch.zeros(shape, device=dev, dtype=deriv_dtype)
            if not value:
                return None, der
        else:
            w = hook.operands.index(wrt)
            der = torch.empty(shape, device=dev, dtype=deriv_dtype)
            if seed is not None:
                seed_op, st = _operand(seed, shape, "seed")
                keep.append(st)
    out_op = _operand(out, shape, "out")[0] if out is not None else None
    der_op = _operand(der, shape, "deriv")[0] if (der is not None and w >= 0) else None
    ref = (lambda o: None if o is None else C.addressof(o))
    shp = (C.c_int32 * 4)(*shape)
    rt.check(rt.lib().af_hook_eval(C.addressof(prog), C.addressof(shp), C.addressof(ops),
                                   len(hook.operands), w,
                                   ref(seed_op), ref(out_op), ref(der_op),
                                   torch.cuda.current_stream(dev).cuda_stream), "af_hook_eval")
    return out, der


def sum_to(t: torch.Tensor, shape) -> torch.Tensor:
    """Sum a [B, H, S, D] derivative over the axes an operand broadcasts on (the reference's
    SUM_TO adjoint, graph.py:575-578)."""
    axes = [i for i in range(4) if shape[i] == 1 and t.shape[i] != 1]
    return t.sum(dim=axes, keepdim=True) if axes else t
