"""Task front-end: DSL text -> which GPU body implements it.

The reference compiles a task through parse_task -> recognize -> build_dag ->
schedule (src/engine.cpp:86-102). The GPU backend needs only the outcome:
whether the statement is one of the bodies it has a fused kernel for, the
operands' roles (A, B, threshold, discount vector) and their orientations.
This module restates just enough of that pipeline:

* a recursive-descent parser for the task grammar (README.md:37-60;
  parser.cpp:142-365): ``where(v in [a..b] and ...) { T[x][y] (+)= expr; }``
  with ``//`` and ``#`` comments;
* the structural recognition conditions 2-4 (recognize.cpp:84-166): three loop
  variables, a 2-D target on two distinct loop variables, exactly one
  ``[i][k]``/``[k][i]`` array (A), one ``[k][j]``/``[j][k]`` array (B), and aux
  leaves that are scalars, ``[i]``, ``[j]`` or ``[i][j]``;
* the body match itself — the statement against the fixed bodies' canonical
  trees after the comparison / product / sum normalisations, else a
  generated body — and the op counts of the reference's compiled program for
  the statement come from the native recogniser (csrc/task.cpp through
  amlt_gpu_recognize), so there is one implementation of the match.

Anything else raises UnsupportedExpression, as the reference does for forms
its vector backend cannot lower.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import _native as N


class TaskError(ValueError):
    pass


# ---------------------------------------------------------------------------
# lexer / parser

_TOK = re.compile(r"\s*(?:(//[^\n]*|#[^\n]*)|(\d+(?:\.\d+)?(?:[eE][-+]?\d+)?)|([A-Za-z_]\w*)|"
                  r"(\+=|==|>=|<=|\.\.|[-+*/<>=()\[\]{};]))")


def _lex(src: str) -> List[str]:
    out, pos = [], 0
    while pos < len(src):
        m = _TOK.match(src, pos)
        if not m or m.end() == pos:
            if src[pos:].strip() == "":
                break
            raise TaskError(f"parse error near {src[pos:pos + 12]!r}")
        pos = m.end()
        if m.group(1):
            continue
        out.append(m.group(2) or m.group(3) or m.group(4))
    return out


# expression trees: ("num", v) | ("ref", name, (idx names...)) | (op, lhs, rhs)
class _Parser:
    def __init__(self, toks):
        self.t = toks
        self.p = 0

    def peek(self):
        return self.t[self.p] if self.p < len(self.t) else None

    def take(self, want=None):
        tok = self.peek()
        if tok is None or (want is not None and tok != want):
            raise TaskError(f"parse error: expected {want!r}, got {tok!r}")
        self.p += 1
        return tok

    def ident(self):
        tok = self.take()
        if not re.match(r"[A-Za-z_]\w*$", tok):
            raise TaskError(f"parse error: expected identifier, got {tok!r}")
        return tok

    def task(self):
        self.take("where")
        self.take("(")
        loops = [self.clause()]
        while self.peek() == "and":
            self.take("and")
            loops.append(self.clause())
        self.take(")")
        self.take("{")
        target = self.ident()
        subs = []
        while self.peek() == "[":
            self.take("[")
            subs.append(self.ident())
            self.take("]")
        op = self.take()
        if op not in ("=", "+="):
            raise TaskError("statement must be `=` or `+=`")
        rhs = self.expr()
        self.take(";")
        self.take("}")
        if self.peek() is not None:
            raise TaskError("trailing input after the task")
        return loops, target, subs, op == "+=", rhs

    def clause(self):
        v = self.ident()
        self.take("in")
        self.take("[")
        lo = self.bound()
        self.take("..")
        hi = self.bound()
        self.take("]")
        return v, lo, hi

    def bound(self):
        tok = self.take()
        return int(tok) if tok.isdigit() else tok

    def expr(self):
        lhs = self.sum()
        if self.peek() in (">", ">=", "<", "<=", "=="):
            op = self.take()
            return (op, lhs, self.sum())
        return lhs

    def sum(self):
        node = self.term()
        while self.peek() in ("+", "-"):
            op = self.take()
            node = (op, node, self.term())
        return node

    def term(self):
        node = self.factor()
        while self.peek() in ("*", "/"):
            op = self.take()
            node = (op, node, self.factor())
        return node

    def factor(self):
        tok = self.peek()
        if tok == "(":
            self.take("(")
            e = self.expr()
            self.take(")")
            return e
        if tok is not None and re.match(r"\d", tok):
            self.take()
            return ("num", float(tok))
        name = self.ident()
        idx = []
        while self.peek() == "[":
            self.take("[")
            idx.append(self.ident())
            self.take("]")
        return ("ref", name, tuple(idx))


# ---------------------------------------------------------------------------
# recognition + body match


@dataclass(frozen=True)
class TaskPlan:
    """What the GPU backend needs from a compiled task."""
    body: int
    body_name: str
    accumulate: bool
    layout_a: int
    layout_b: int
    thres_class: int
    thres_value: float
    a_name: str
    b_name: str
    result_name: str
    thres_name: Optional[str]
    dis_name: Optional[str]
    var_i: str
    var_j: str
    var_k: str
    dims: Tuple[str, str, str]  # range-end identifiers bound to (M, K, N)
    # generic statements (BODY_GENERIC): aux leaves in first-use order, their
    # index classes (N.LEAF_*), the source the native planner compiles
    aux_names: Tuple[str, ...] = ()
    aux_classes: Tuple[int, ...] = ()
    source: str = ""
    # the reference's compiled program for the statement: instructions per
    # opcode, and its body-op flops per inner iteration
    program: Dict[str, int] = field(default_factory=dict, compare=False, hash=False)
    program_flops: int = 0


_BODY_NAMES = {N.BODY_GEMM: "gemm", N.BODY_DISCOUNT: "discount", N.BODY_BOOST: "boost",
               N.BODY_SQDIFF: "sqdiff", N.BODY_EQCOUNT: "eqcount", N.BODY_THRCOUNT: "thrcount",
               N.BODY_GENERIC: "generic"}


def compile_task(source: str) -> TaskPlan:
    """Parses and recognises a task; raises UnsupportedExpression (from
    engine) when it is not one of the GPU bodies."""
    from .engine import UnsupportedExpression

    loops, target, subs, accumulate, rhs = _Parser(_lex(source)).task()
    var_names = [v for v, _, _ in loops]
    if len(loops) != 3:
        raise UnsupportedExpression("not an MMLT: needs exactly three loop variables")
    if len(subs) != 2 or subs[0] == subs[1] or any(s not in var_names for s in subs):
        raise UnsupportedExpression("not an MMLT: target must be 2-D over two distinct loop variables")
    vi, vj = subs
    vk = next(v for v in var_names if v not in subs)
    ends = {v: hi for v, _, hi in loops}
    starts = {v: lo for v, lo, _ in loops}
    if any(starts[v] != 0 for v in var_names):
        raise UnsupportedExpression("loop ranges must start at 0 for the GPU backend")

    roles = {}  # name -> ("A"|"B", layout) or ("aux", cls)

    def classify(node):
        k = node[0]
        if k == "num":
            return node
        if k == "ref":
            name, idx = node[1], node[2]
            if name == target:
                raise UnsupportedExpression("target appears on the right-hand side")
            if not idx:
                if name in var_names:
                    raise UnsupportedExpression("loop variable used as a value")
                return ("aux", name, "c")
            if any(x not in var_names for x in idx):
                raise UnsupportedExpression("subscripts must be loop variables")
            if idx == (vi, vk) or idx == (vk, vi):
                role = ("A", N.LAYOUT_NORMAL if idx == (vi, vk) else N.LAYOUT_TRANSPOSED)
            elif idx == (vk, vj) or idx == (vj, vk):
                role = ("B", N.LAYOUT_NORMAL if idx == (vk, vj) else N.LAYOUT_TRANSPOSED)
            elif idx == (vi,):
                role = ("aux", "i")
            elif idx == (vj,):
                role = ("aux", "j")
            elif idx == (vi, vj):
                role = ("aux", "ij")
            else:
                raise UnsupportedExpression(f"operand {name}{list(idx)} does not fit the MMLT pattern")
            prev = roles.get(name)
            if prev is not None and prev != role:
                raise UnsupportedExpression(f"array {name} used with two index patterns")
            roles[name] = role
            if role[0] in ("A", "B"):
                return ("role", role[0])
            return ("aux", name, role[1])
        return (k, classify(node[1]), classify(node[2]))

    tree = classify(rhs)
    a_names = [n for n, r in roles.items() if r[0] == "A"]
    b_names = [n for n, r in roles.items() if r[0] == "B"]
    if len(a_names) != 1 or len(b_names) != 1:
        raise UnsupportedExpression("not an MMLT: needs exactly one A[i][k] and one B[k][j] array")

    # The body match (six fixed bodies after the canonical rewrites, else a
    # generated body), the leaf roles and the reference program's op counts
    # come from the native recogniser (csrc/task.cpp, amlt_gpu_recognize).
    import ctypes as C
    info = N.TaskInfoC()
    st = N.lib().amlt_gpu_recognize(source.encode(), C.byref(info))
    if st != N.OK:
        msg = N.lib().amlt_gpu_last_error(None)
        raise UnsupportedExpression(msg.decode() if msg else "statement not recognised")
    d = info.desc
    names = tuple(info.aux_names[q].value.decode() for q in range(info.n_aux))
    thres = info.thres.decode() or None
    dis = info.dis.decode() or None
    program = {op: int(info.prog_counts[c]) for c, op in enumerate(N.PROG_OPCODES) if info.prog_counts[c]}
    return TaskPlan(
        body=d.body, body_name=_BODY_NAMES[d.body], accumulate=bool(d.accumulate),
        layout_a=d.layout_a, layout_b=d.layout_b, thres_class=d.thres_class,
        thres_value=d.thres_value, a_name=info.a.decode(), b_name=info.b.decode(),
        result_name=target, thres_name=thres, dis_name=dis, var_i=vi, var_j=vj, var_k=vk,
        dims=(str(ends[vi]), str(ends[vk]), str(ends[vj])),
        aux_names=names if d.body == N.BODY_GENERIC else (),
        aux_classes=tuple(int(info.aux_class[q]) for q in range(info.n_aux)) if d.body == N.BODY_GENERIC else (),
        source=source, program=program, program_flops=int(info.prog_flops))


# ---------------------------------------------------------------------------
# built-in task names (presets.hpp / src/presets.cpp:8-94): matmul, q1, q2, q3
# with an optional threshold suffix (-tc | -ti | -tj | -tij; q1/q2 default
# -tj, q3 default -tc, none for matmul) and an optional orientation suffix
# (-ab | -atb | -abt | -atbt), in any order, each at most once.

_PRESET_BASES = ("matmul", "q1", "q2", "q3")
_THRES_FORMS = {"tc": "100", "ti": "thres[i]", "tj": "thres[j]", "tij": "thres[i][j]"}
_ORIENTS = ("ab", "atb", "abt", "atbt")


def preset_names() -> List[str]:
    """Every accepted built-in name with explicit suffixes (the 52 of
    presets.cpp: 4 matmul orientations + 3 bases x 4 thresholds x 4)."""
    out = [f"matmul-{o}" for o in _ORIENTS]
    for base in ("q1", "q2", "q3"):
        out += [f"{base}-{t}-{o}" for t in _THRES_FORMS for o in _ORIENTS]
    return out


def preset_source(name: str) -> Optional[str]:
    """DSL text of a built-in task, or None for an unknown name."""
    parts = name.split("-")
    base = parts[0]
    if base not in _PRESET_BASES:
        return None
    thres = "tc" if base == "q3" else "tj"
    orient = "ab"
    seen_t = seen_o = False
    for s in parts[1:]:
        if s in _THRES_FORMS and not seen_t and base != "matmul":
            thres, seen_t = s, True
        elif s in _ORIENTS and not seen_o:
            orient, seen_o = s, True
        else:
            return None
    a = "A[k][i]" if orient in ("atb", "atbt") else "A[i][k]"
    b = "B[j][k]" if orient in ("abt", "atbt") else "B[k][j]"
    ab = f"{a}*{b}"
    t = _THRES_FORMS[thres]
    rhs = {"matmul": ab,
           "q1": f"{ab} - ({ab} > {t})*{ab}*dis[j]",
           "q2": f"{ab} + ({ab} > {t})*({ab} - {t})",
           "q3": f"({ab} > {t})"}[base]
    return ("where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
            f"  R[i][j] += {rhs};\n}}\n")
