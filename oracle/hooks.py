"""Hook expressions on numpy float64 arrays (oracle side; TEST INFRASTRUCTURE ONLY).

The hook language (attnforge ``exprlang.py:1-19``) is a syntactic subset of Python expressions,
so the oracle parses with :mod:`ast` and walks the tree — deliberately independent of the product
parser (``paper_2502_15349_b200/hooklang.py``) so the two cross-check each other.

``evaluate`` follows ``engine.eval_expr`` / ``engine._eval`` (engine.py:138-179): IEEE semantics,
``log(0) = -inf``, row reductions over the last axis with ascending accumulation
(engine.py:83-101).  ``evaluate_dual`` carries a derivative with respect to one variable, using
the reference's adjoint rules (graph.py:481-569): max/min ties route to the first operand, where()
routes by branch, clamp passes the gradient inside the closed interval, abs/abssum use
sign(0) = +1, relu is max(x, 0) (tie → x).
"""

from __future__ import annotations

import ast
import math
from functools import lru_cache

import numpy as np

_ERR = dict(divide="ignore", invalid="ignore", over="ignore", under="ignore")


@lru_cache(maxsize=None)
def compile_hook(src: str) -> ast.expr:
    tree = ast.parse(src.strip(), mode="eval").body
    for node in ast.walk(tree):
        if isinstance(node, ast.Compare) and len(node.ops) != 1:
            raise ValueError(f"chained comparison in hook {src!r}")
    return tree


def row_sum(x):
    x = np.asarray(x, np.float64)
    out = np.zeros(x.shape[:-1] + (1,))
    for t in range(x.shape[-1]):
        out[..., 0] += x[..., t]
    return out


def row_abssum(x):
    return row_sum(np.abs(np.asarray(x, np.float64)))


def row_max(x):
    return np.max(np.asarray(x, np.float64), axis=-1, keepdims=True)


def _sig(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, np.float64)))


_UN = {"exp": np.exp, "exp2": np.exp2, "log": np.log, "abs": np.abs, "tanh": np.tanh,
       "sigmoid": _sig, "relu": lambda x: np.maximum(x, 0.0), "sqrt": np.sqrt,
       "reduceSum": row_sum, "reduceMax": row_max, "reduceAbssum": row_abssum}
_BIN = {ast.Add: np.add, ast.Sub: np.subtract, ast.Mult: np.multiply, ast.Div: np.divide}
_CMP = {ast.Eq: np.equal, ast.NotEq: np.not_equal, ast.Lt: np.less, ast.LtE: np.less_equal,
        ast.Gt: np.greater, ast.GtE: np.greater_equal}


def evaluate(src: str, env: dict):
    with np.errstate(**_ERR):
        return _ev(compile_hook(src), env)


def _ev(n, env):
    if isinstance(n, ast.Constant):
        return float(n.value)
    if isinstance(n, ast.Name):
        if n.id == "inf":
            return math.inf
        return env[n.id]
    if isinstance(n, ast.UnaryOp) and isinstance(n.op, ast.USub):
        return -_ev(n.operand, env)
    if isinstance(n, ast.BinOp):
        return _BIN[type(n.op)](np.float64(1) * _ev(n.left, env), _ev(n.right, env))
    if isinstance(n, ast.Compare):
        return _CMP[type(n.ops[0])](_ev(n.left, env), _ev(n.comparators[0], env)).astype(
            np.float64)
    if isinstance(n, ast.Call):
        f = n.func.id
        a = [_ev(x, env) for x in n.args]
        if f in _UN:
            return _UN[f](a[0])
        if f == "max":
            return np.maximum(a[0], a[1])
        if f == "min":
            return np.minimum(a[0], a[1])
        if f == "clamp":
            return np.clip(a[0], a[1], a[2])
        if f == "where":
            return np.where(np.asarray(a[0]) != 0, a[1], a[2])
    raise ValueError(f"unsupported hook node {ast.dump(n)}")


def evaluate_dual(src: str, env: dict, wrt: str, seed=1.0):
    """(value, d value / d env[wrt]) for an elementwise hook (no row reductions)."""
    with np.errstate(**_ERR):
        return _dv(compile_hook(src), env, wrt, seed)


def _dv(n, env, wrt, seed):
    if isinstance(n, ast.Constant):
        return float(n.value), 0.0
    if isinstance(n, ast.Name):
        if n.id == "inf":
            return math.inf, 0.0
        v = env[n.id]
        return v, (seed if n.id == wrt else 0.0)
    if isinstance(n, ast.UnaryOp) and isinstance(n.op, ast.USub):
        v, d = _dv(n.operand, env, wrt, seed)
        return -v, -d
    if isinstance(n, ast.BinOp):
        a, da = _dv(n.left, env, wrt, seed)
        b, db = _dv(n.right, env, wrt, seed)
        a = np.float64(1) * a
        if isinstance(n.op, ast.Add):
            return a + b, da + db
        if isinstance(n.op, ast.Sub):
            return a - b, da - db
        if isinstance(n.op, ast.Mult):
            return a * b, da * b + a * db
        q = a / b
        return q, da / b - q * db / b
    if isinstance(n, ast.Compare):
        return _ev(n, env), 0.0
    if isinstance(n, ast.Call):
        f = n.func.id
        if f == "where":
            c = np.asarray(_ev(n.args[0], env)) != 0
            a, da = _dv(n.args[1], env, wrt, seed)
            b, db = _dv(n.args[2], env, wrt, seed)
            return np.where(c, a, b), np.where(c, da, db)
        if f == "sqrt":
            return np.sqrt(_ev(n.args[0], env)), 0.0
        args = [_dv(x, env, wrt, seed) for x in n.args]
        (x, dx) = args[0]
        if f == "exp":
            y = np.exp(x)
            return y, y * dx
        if f == "exp2":
            y = np.exp2(x)
            return y, y * math.log(2.0) * dx
        if f == "log":
            return np.log(x), dx / x
        if f == "abs":
            return np.abs(x), np.where(np.asarray(x) >= 0, 1.0, -1.0) * dx
        if f == "tanh":
            y = np.tanh(x)
            return y, (1.0 - y * y) * dx
        if f == "sigmoid":
            y = _sig(x)
            return y, y * (1.0 - y) * dx
        if f == "relu":
            return np.maximum(x, 0.0), np.where(np.asarray(x) >= 0.0, 1.0, 0.0) * dx
        if f in ("max", "min"):
            (y, dy) = args[1]
            first = (np.asarray(x) >= y) if f == "max" else (np.asarray(x) <= y)
            return (np.maximum(x, y) if f == "max" else np.minimum(x, y)), \
                np.where(first, dx, dy)
        if f == "clamp":
            lo, hi = args[1][0], args[2][0]
            inside = (np.asarray(x) >= lo) & (np.asarray(x) <= hi)
            return np.clip(x, lo, hi), np.where(inside, dx, 0.0)
    raise ValueError(f"hook node not differentiable elementwise: {ast.dump(n)}")


def free_names(src: str) -> set[str]:
    return {n.id for n in ast.walk(compile_hook(src)) if isinstance(n, ast.Name)} - {"inf"}
