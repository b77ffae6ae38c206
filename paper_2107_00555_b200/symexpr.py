"""Symbolic integer expressions used by map ranges, memlet subsets and shapes.

The serialized graph (schema v1, reference pkg/src/sdfgkit/serialize.py:1-16)
stores every size, range and subset as text in the grammar of
pkg/src/sdfgkit/symbolic.py:758-891 (``+ - * //``, unary minus, ``min``/``max``,
integer literals, names).  This module parses that text into a small tuple
tree and offers what the B200 planner needs:

* ``evaluate`` — exact Python-int evaluation (floor division rounds toward
  -inf like symbolic.py:196-199),
* ``affine`` — decomposition into ``c0 + sum(c_i * p_i)`` over chosen names
  after concrete symbol substitution (the planner works with concrete
  bindings), used for fusion legality and bounds checks,
* ``interval`` — conservative value range over boxed parameter ranges,
* ``to_c`` — int64 C text for generated device code.

Subsets keep the reference's inclusive-end convention: ``b:e:s`` covers
``range(b, e + 1, s)`` (symbolic.py:549-556).
"""

from __future__ import annotations

import re
from typing import Mapping

# Node encoding: ("c", int) | ("s", name) | (op, left, right) with op in
# {"+", "-", "*", "//", "min", "max"}.

_TOKEN = re.compile(r"\s*(\d+|[A-Za-z_][A-Za-z_0-9]*|//|[-+*(),:])")


class ExprError(ValueError):
    pass


class _P:
    def __init__(self, text: str):
        self.toks: list[str] = []
        pos = 0
        while pos < len(text):
            m = _TOKEN.match(text, pos)
            if not m:
                if text[pos:].strip():
                    raise ExprError(f"bad symbolic expression near {text[pos:]!r}")
                break
            self.toks.append(m.group(1))
            pos = m.end()
        self.i = 0

    def peek(self):
        return self.toks[self.i] if self.i < len(self.toks) else None

    def take(self, want=None):
        t = self.peek()
        if t is None:
            raise ExprError("unexpected end of symbolic expression")
        if want is not None and t != want:
            raise ExprError(f"expected {want!r}, got {t!r}")
        self.i += 1
        return t

    def parse(self):
        e = self.addsub()
        if self.peek() is not None:
            raise ExprError(f"trailing tokens {self.toks[self.i:]}")
        return e

    def addsub(self):
        e = self.muldiv()
        while self.peek() in ("+", "-"):
            op = self.take()
            e = (op, e, self.muldiv())
        return e

    def muldiv(self):
        e = self.unary()
        while self.peek() in ("*", "//"):
            op = self.take()
            e = (op, e, self.unary())
        return e

    def unary(self):
        if self.peek() == "-":
            self.take()
            return ("*", ("c", -1), self.unary())
        if self.peek() == "+":
            self.take()
            return self.unary()
        return self.atom()

    def atom(self):
        t = self.take()
        if t.isdigit():
            return ("c", int(t))
        if t == "(":
            e = self.addsub()
            self.take(")")
            return e
        if t in ("min", "max"):
            self.take("(")
            a = self.addsub()
            self.take(",")
            b = self.addsub()
            self.take(")")
            return (t, a, b)
        if re.fullmatch(r"[A-Za-z_][A-Za-z_0-9]*", t):
            return ("s", t)
        raise ExprError(f"unexpected token {t!r}")


_cache: dict[str, tuple] = {}


def parse(text) -> tuple:
    if isinstance(text, int):
        return ("c", int(text))
    text = str(text)
    e = _cache.get(text)
    if e is None:
        e = _P(text).parse()
        _cache[text] = e
    return e


def const(v: int) -> tuple:
    return ("c", int(v))


def sym(name: str) -> tuple:
    return ("s", name)


def free_symbols(e) -> set[str]:
    out: set[str] = set()

    def walk(x):
        if x[0] == "s":
            out.add(x[1])
        elif x[0] != "c":
            walk(x[1])
            walk(x[2])

    walk(e)
    return out


def evaluate(e, env: Mapping[str, int]) -> int:
    k = e[0]
    if k == "c":
        return e[1]
    if k == "s":
        try:
            return int(env[e[1]])
        except KeyError:
            raise KeyError(f"unbound symbol '{e[1]}'") from None
    a = evaluate(e[1], env)
    b = evaluate(e[2], env)
    if k == "+":
        return a + b
    if k == "-":
        return a - b
    if k == "*":
        return a * b
    if k == "//":
        if b == 0:
            raise ZeroDivisionError("symbolic floor division by zero")
        return a // b
    if k == "min":
        return min(a, b)
    if k == "max":
        return max(a, b)
    raise ExprError(f"bad node {k}")


def substitute(e, env: Mapping[str, int]):
    """Replace bound names by constants and fold constant subtrees."""
    k = e[0]
    if k == "c":
        return e
    if k == "s":
        return ("c", int(env[e[1]])) if e[1] in env else e
    a = substitute(e[1], env)
    b = substitute(e[2], env)
    if a[0] == "c" and b[0] == "c":
        return ("c", evaluate((k, a, b), {}))
    return (k, a, b)


def affine(e, params: tuple[str, ...] | list[str], env: Mapping[str, int]):
    """Return (c0, {p: c}) if ``e`` is affine in ``params`` once every other
    name is replaced by its value from ``env``; otherwise None."""
    k = e[0]
    if k == "c":
        return e[1], {}
    if k == "s":
        if e[1] in params:
            return 0, {e[1]: 1}
        if e[1] in env:
            return int(env[e[1]]), {}
        return None
    a = affine(e[1], params, env)
    b = affine(e[2], params, env)
    if a is None or b is None:
        return None
    if k in ("+", "-"):
        sgn = 1 if k == "+" else -1
        co = dict(a[1])
        for p, c in b[1].items():
            co[p] = co.get(p, 0) + sgn * c
        return a[0] + sgn * b[0], {p: c for p, c in co.items() if c != 0}
    if k == "*":
        if not a[1]:
            return a[0] * b[0], {p: a[0] * c for p, c in b[1].items() if a[0] * c}
        if not b[1]:
            return a[0] * b[0], {p: b[0] * c for p, c in a[1].items() if b[0] * c}
        return None
    if k in ("//", "min", "max"):
        if not a[1] and not b[1]:
            return evaluate((k, ("c", a[0]), ("c", b[0])), {}), {}
        return None
    return None


def interval(e, box: Mapping[str, tuple[int, int]], env: Mapping[str, int]):
    """Conservative [lo, hi] of ``e`` with names in ``box`` ranging over their
    closed intervals and other names fixed by ``env``."""
    k = e[0]
    if k == "c":
        return e[1], e[1]
    if k == "s":
        if e[1] in box:
            return box[e[1]]
        v = int(env[e[1]])
        return v, v
    a0, a1 = interval(e[1], box, env)
    b0, b1 = interval(e[2], box, env)
    if k == "+":
        return a0 + b0, a1 + b1
    if k == "-":
        return a0 - b1, a1 - b0
    if k == "*":
        c = (a0 * b0, a0 * b1, a1 * b0, a1 * b1)
        return min(c), max(c)
    if k == "//":
        if b0 <= 0 <= b1:
            raise ZeroDivisionError("possible symbolic division by zero")
        c = (a0 // b0, a0 // b1, a1 // b0, a1 // b1)
        return min(c), max(c)
    if k == "min":
        return min(a0, b0), min(a1, b1)
    if k == "max":
        return max(a0, b0), max(a1, b1)
    raise ExprError(f"bad node {k}")


def to_c(e, name_of=lambda n: n) -> str:
    """int64 C expression; ``name_of`` maps a symbol/param name to C text."""
    k = e[0]
    if k == "c":
        return f"{e[1]}LL" if e[1] >= 0 else f"({e[1]}LL)"
    if k == "s":
        return name_of(e[1])
    a = to_c(e[1], name_of)
    b = to_c(e[2], name_of)
    if k in ("+", "-", "*"):
        return f"({a} {k} {b})"
    if k == "//":
        return f"b2_floordiv_ll({a}, {b})"
    if k == "min":
        return f"b2_min_ll({a}, {b})"
    if k == "max":
        return f"b2_max_ll({a}, {b})"
    raise ExprError(f"bad node {k}")


def to_text(e) -> str:
    k = e[0]
    if k == "c":
        return str(e[1])
    if k == "s":
        return e[1]
    if k in ("min", "max"):
        return f"{k}({to_text(e[1])}, {to_text(e[2])})"
    return f"({to_text(e[1])} {k} {to_text(e[2])})"


def to_py(e, name_of=lambda n: n) -> str:
    """Python source text (used to compile fast per-launch argument builders)."""
    k = e[0]
    if k == "c":
        return f"({e[1]})"
    if k == "s":
        return name_of(e[1])
    a = to_py(e[1], name_of)
    b = to_py(e[2], name_of)
    if k in ("+", "-", "*", "//"):
        return f"({a} {k} {b})"
    return f"{k}({a}, {b})"


def split_top(text: str, sep: str) -> list[str]:
    parts, depth, cur = [], 0, []
    for ch in text:
        if ch == "(":
            depth += 1
        elif ch == ")":
            depth -= 1
        if ch == sep and depth == 0:
            parts.append("".join(cur))
            cur = []
        else:
            cur.append(ch)
    parts.append("".join(cur))
    return parts


def parse_subset(text: str) -> list[tuple[tuple, tuple, tuple]]:
    """``"b:e:s, b2:e2"`` -> [(b, e, s), ...] with inclusive ends."""
    text = text.strip()
    if not text:
        return []
    dims = []
    for part in split_top(text, ","):
        pieces = split_top(part, ":")
        if len(pieces) == 1:
            b = parse(pieces[0])
            dims.append((b, b, ("c", 1)))
        elif len(pieces) == 2:
            dims.append((parse(pieces[0]), parse(pieces[1]), ("c", 1)))
        elif len(pieces) == 3:
            dims.append(tuple(parse(p) for p in pieces))
        else:
            raise ExprError(f"bad subset dimension {part!r}")
    return dims


def eval_subset(dims, env: Mapping[str, int]) -> list[range]:
    out = []
    for b, e, s in dims:
        bv, ev, sv = evaluate(b, env), evaluate(e, env), evaluate(s, env)
        if sv < 1:
            raise ValueError(f"stride {sv} < 1 in subset")
        out.append(range(bv, ev + 1, sv))
    return out
