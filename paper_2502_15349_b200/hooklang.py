"""Hook expression language (score_mod / mask_mod / online_func / feature_map / decay hooks).

Accepts exactly the language of the reference (attnforge ``exprlang.py:1-19``, grammar
``exprlang.py:151-254``; documented in ``docs/expression-language.md``):

* literals (``1``, ``2.5e-3``), names, ``inf``; binary ``+ - * /`` with the usual precedence and
  unary minus binding tighter than ``*``; comparisons only as the condition of ``where``;
* functions ``exp exp2 log abs tanh sigmoid relu sqrt`` (1 arg), ``max min`` (2), ``clamp where``
  (3), and the row reductions ``reduceSum reduceMax reduceAbssum``;
* ``sqrt`` folds at lowering time on a literal or named constant; division by a literal zero is a
  parse error.

The AST is a small set of frozen dataclasses.  Besides parsing and printing this module offers
``const_value`` (compile-time folding against the dims environment) and ``fold`` (partial
evaluation), which the lowering (``plan.py``) uses to classify hooks into kernel families.
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass

from .errors import LowerError, ParseError


@dataclass(frozen=True, slots=True)
class Num:
    value: float


@dataclass(frozen=True, slots=True)
class Name:
    name: str


@dataclass(frozen=True, slots=True)
class Neg:
    operand: "Node"


@dataclass(frozen=True, slots=True)
class BinOp:
    op: str  # + - * /
    lhs: "Node"
    rhs: "Node"


@dataclass(frozen=True, slots=True)
class Cmp:
    op: str  # == != < <= > >=
    lhs: "Node"
    rhs: "Node"


@dataclass(frozen=True, slots=True)
class Fn:
    func: str
    args: tuple


Node = Num | Name | Neg | BinOp | Cmp | Fn

ARITY = {
    "exp": 1, "exp2": 1, "log": 1, "abs": 1, "tanh": 1, "sigmoid": 1, "relu": 1, "sqrt": 1,
    "reduceSum": 1, "reduceMax": 1, "reduceAbssum": 1,
    "max": 2, "min": 2, "clamp": 3, "where": 3,
}
REDUCTIONS = frozenset({"reduceSum", "reduceMax", "reduceAbssum"})
CMP_OPS = ("==", "!=", "<=", ">=", "<", ">")

_TOKEN = re.compile(r"""
    (?P<ws>\s+)
  | (?P<badexp>(?:\d+\.?\d*|\.\d+)[eE](?:[+-](?!\d)|(?![+\-\d])))
  | (?P<num>(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)
  | (?P<name>[A-Za-z_][A-Za-z0-9_]*)
  | (?P<op>==|!=|<=|>=|[-+*/(),<>])
""", re.VERBOSE)


def _lex(src: str) -> list[tuple[str, str, int]]:
    out: list[tuple[str, str, int]] = []
    pos = 0
    while pos < len(src):
        m = _TOKEN.match(src, pos)
        if m is None:
            raise ParseError(f"unexpected character {src[pos]!r}", offset=pos)
        kind = m.lastgroup
        if kind == "badexp":
            raise ParseError("malformed exponent", offset=pos)
        if kind != "ws":
            out.append((kind, m.group(), pos))
        pos = m.end()
    out.append(("end", "", len(src)))
    return out


class _Reader:
    """Recursive-descent reader over the token list (precedence climbing by level)."""

    def __init__(self, src: str):
        self.toks = _lex(src)
        self.i = 0

    def peek(self):
        return self.toks[self.i]

    def take(self):
        t = self.toks[self.i]
        self.i += 1
        return t

    def want(self, text: str):
        kind, val, off = self.take()
        if kind == "end" or val != text:
            raise ParseError(f"expected {text!r}", offset=off)

    def expr(self) -> Node:
        lhs = self.sum()
        kind, val, off = self.peek()
        if kind == "op" and val in CMP_OPS:
            self.take()
            rhs = self.sum()
            k2, v2, o2 = self.peek()
            if k2 == "op" and v2 in CMP_OPS:
                raise ParseError("chained comparisons are not supported", offset=o2)
            return Cmp(val, lhs, rhs)
        return lhs

    def sum(self) -> Node:
        node = self.product()
        while self.peek()[0] == "op" and self.peek()[1] in "+-":
            op = self.take()[1]
            node = BinOp(op, node, self.product())
        return node

    def product(self) -> Node:
        node = self.unary()
        while self.peek()[0] == "op" and self.peek()[1] in "*/":
            _, op, off = self.take()
            rhs = self.unary()
            if op == "/" and isinstance(rhs, Num) and rhs.value == 0.0:
                raise ParseError("division by zero literal", offset=off)
            node = BinOp(op, node, rhs)
        return node

    def unary(self) -> Node:
        if self.peek()[:2] == ("op", "-"):
            self.take()
            inner = self.unary()
            return Num(-inner.value) if isinstance(inner, Num) else Neg(inner)
        return self.atom()

    def atom(self) -> Node:
        kind, val, off = self.take()
        if kind == "num":
            return Num(float(val))
        if kind == "name" and val in ARITY:
            self.want("(")
            args = [self.expr()]
            while self.peek()[:2] == ("op", ","):
                self.take()
                args.append(self.expr())
            self.want(")")
            if len(args) != ARITY[val]:
                raise ParseError(f"{val} takes {ARITY[val]} argument(s), got {len(args)}",
                                 offset=off)
            return Fn(val, tuple(args))
        if kind == "name":
            return Num(math.inf) if val == "inf" else Name(val)
        if (kind, val) == ("op", "("):
            inner = self.expr()
            self.want(")")
            return inner
        raise ParseError("expected an expression", offset=off)


def parse(src: str) -> Node:
    """Parse one hook expression; ``ParseError`` carries the byte offset of the problem."""
    r = _Reader(src)
    node = r.expr()
    kind, _, off = r.peek()
    if kind != "end":
        raise ParseError("trailing input after expression", offset=off)
    return node


# ───────────────────────────── printing / inspection ─────────────────────────────

def _num_text(v: float) -> str:
    if v == math.inf:
        return "inf"
    if v == -math.inf:
        return "-inf"
    if v == int(v) and abs(v) < 1e16:
        return str(int(v))
    return repr(v)


def to_source(node: Node, level: int = 0) -> str:
    """Render with minimal parentheses; ``parse(to_source(parse(s))) == parse(s)``."""
    if isinstance(node, Num):
        t = _num_text(node.value)
        own = 3 if t.startswith("-") else 4
        return f"({t})" if own < level else t
    if isinstance(node, Name):
        return node.name
    if isinstance(node, Fn):
        return f"{node.func}({', '.join(to_source(a, 0) for a in node.args)})"
    if isinstance(node, Neg):
        body = "-" + to_source(node.operand, 3)
        return f"({body})" if 3 < level else body
    if isinstance(node, BinOp):
        own = 1 if node.op in "+-" else 2
        body = f"{to_source(node.lhs, own)} {node.op} {to_source(node.rhs, own + 1)}"
        return f"({body})" if own < level else body
    if isinstance(node, Cmp):
        body = f"{to_source(node.lhs, 1)} {node.op} {to_source(node.rhs, 1)}"
        return f"({body})" if 0 < level else body
    raise TypeError(f"not a hook expression: {node!r}")


def free_names(node: Node) -> set[str]:
    if isinstance(node, Name):
        return {node.name}
    if isinstance(node, Neg):
        return free_names(node.operand)
    if isinstance(node, (BinOp, Cmp)):
        return free_names(node.lhs) | free_names(node.rhs)
    if isinstance(node, Fn):
        out: set[str] = set()
        for a in node.args:
            out |= free_names(a)
        return out
    return set()


def calls(node: Node) -> set[str]:
    """Function names used anywhere in the expression."""
    if isinstance(node, Fn):
        out = {node.func}
        for a in node.args:
            out |= calls(a)
        return out
    if isinstance(node, Neg):
        return calls(node.operand)
    if isinstance(node, (BinOp, Cmp)):
        return calls(node.lhs) | calls(node.rhs)
    return set()


def check_elementwise(node: Node, where: str) -> None:
    """Reject row reductions / stray comparisons in an elementwise-only position
    (exprlang.py:347-357, 383-386)."""
    if isinstance(node, Cmp):
        raise LowerError("comparisons are only allowed inside where()", hook=where)

    def walk(n: Node, in_where_cond: bool) -> None:
        if isinstance(n, Cmp) and not in_where_cond:
            raise LowerError("comparisons are only allowed inside where()", hook=where)
        if isinstance(n, Fn):
            if n.func in REDUCTIONS:
                raise LowerError(f"{n.func} is not allowed in an elementwise-only position",
                                 hook=where)
            if n.func == "where" and not isinstance(n.args[0], Cmp):
                raise LowerError("where() condition must be a comparison", hook=where)
            for k, a in enumerate(n.args):
                walk(a, n.func == "where" and k == 0)
        elif isinstance(n, Cmp):
            walk(n.lhs, False)
            walk(n.rhs, False)
        elif isinstance(n, BinOp):
            walk(n.lhs, False)
            walk(n.rhs, False)
        elif isinstance(n, Neg):
            walk(n.operand, False)

    walk(node, False)


def const_value(node: Node, env: dict[str, float]) -> float | None:
    """Compile-time value when the expression only involves literals and constants in ``env``
    (e.g. the dims constants ``dimqk``/``seqk``); ``None`` otherwise."""
    v = fold(node, env)
    return v.value if isinstance(v, Num) else None


_UNARY = {
    "exp": math.exp, "exp2": lambda x: 2.0 ** x, "abs": abs, "tanh": math.tanh,
    "sigmoid": lambda x: 1.0 / (1.0 + math.exp(-x)) if x > -700 else 0.0,
    "relu": lambda x: max(x, 0.0),
}


def _safe(fn, *a) -> float | None:
    try:
        return float(fn(*a))
    except (OverflowError, ValueError, ZeroDivisionError):
        return None


def fold(node: Node, env: dict[str, float]) -> Node:
    """Partially evaluate constant sub-expressions against ``env`` (IEEE semantics for log(0),
    x/0)."""
    if isinstance(node, Name):
        return Num(float(env[node.name])) if node.name in env else node
    if isinstance(node, Num):
        return node
    if isinstance(node, Neg):
        inner = fold(node.operand, env)
        return Num(-inner.value) if isinstance(inner, Num) else Neg(inner)
    if isinstance(node, (BinOp, Cmp)):
        a, b = fold(node.lhs, env), fold(node.rhs, env)
        if isinstance(a, Num) and isinstance(b, Num):
            x, y = a.value, b.value
            if isinstance(node, BinOp):
                if node.op == "+":
                    return Num(x + y)
                if node.op == "-":
                    return Num(x - y)
                if node.op == "*":
                    return Num(x * y)
                if y == 0.0:
                    return Num(math.copysign(math.inf, x) if x != 0 else math.nan)
                return Num(x / y)
            res = {"==": x == y, "!=": x != y, "<": x < y, "<=": x <= y, ">": x > y,
                   ">=": x >= y}[node.op]
            return Num(1.0 if res else 0.0)
        return type(node)(node.op, a, b)
    if isinstance(node, Fn):
        args = tuple(fold(a, env) for a in node.args)
        if all(isinstance(a, Num) for a in args) and node.func not in REDUCTIONS:
            vals = [a.value for a in args]
            if node.func == "log":
                x = vals[0]
                r = -math.inf if x == 0 else (_safe(math.log, x) if x > 0 else math.nan)
            elif node.func == "sqrt":
                r = _safe(math.sqrt, vals[0])
            elif node.func in _UNARY:
                r = _safe(_UNARY[node.func], vals[0])
            elif node.func == "max":
                r = max(vals)
            elif node.func == "min":
                r = min(vals)
            elif node.func == "clamp":
                r = min(max(vals[0], vals[1]), vals[2])
            elif node.func == "where":
                r = vals[1] if vals[0] != 0 else vals[2]
            else:
                r = None
            if r is not None:
                return Num(r)
        return Fn(node.func, args)
    raise TypeError(f"not a hook expression: {node!r}")
