"""ImgQL front end: text -> hash-consed task DAG.

Host layer (not the hot path).  It mirrors the reference front end so the
task graphs handed to the device program are node-for-node the reference's:

* ``tokenize``  -- proj/src/lexer.cpp:27-121 (`//` comments, longest-match
  operators, strtod numbers, keywords let/load/save/print/import);
* ``parse``     -- proj/src/parser.cpp:15-184 (commands; 5 left-associative
  infix levels, ast.cpp:12-19; prefix ``!``; application);
* ``expand``    -- proj/src/task_graph.cpp:131-362 (builtin arity table,
  by-name macro substitution in the caller's scope, ``intern`` hash-consing
  so dependencies always have smaller ids, imports processed once).

The builtin table gains two opcodes the reference lacks: ``maxvol`` and
``components`` (the ccl::label image of a mask, saved as an RGB label PNG),
both of arity 1.
"""
from __future__ import annotations

import math
import re
import struct
from dataclasses import dataclass, field
from typing import Callable, Optional, Union

# proj/stdlib/stdlib.imgql:5-14 -- the four derived operators (the spec's
# definitions of interior/touch/grow/surrounded).
STDLIB = """// Standard library: derived spatial operators over near and reach.
let interior(a) = !near(!a)
let touch(a,b) = a & reach(b,a)
let grow(a,b) = a | touch(b,a)
let surrounded(a,b) = a & !reach(!(a|b), !b)
"""


class SpecError(Exception):
    """Lexical / syntax / expansion error (errors.hpp:18-50); CLI exit code 1."""

    def __init__(self, stage: str, message: str, pos: tuple[int, int] = (0, 0)):
        name = {"lex": "lexical error", "parse": "syntax error", "expand": "expansion error"}[stage]
        where = f" at {pos[0]}:{pos[1]}" if pos[0] > 0 else ""
        super().__init__(f"{name}{where}: {message}")
        self.stage, self.pos, self.raw = stage, pos, message


# ---------------------------------------------------------------- lexer
_KEYWORDS = {"let", "load", "save", "print", "import"}
_OPS = [">=.", "<=.", ">.", "<.", "=.", "!", "&", "|", "+", "-", "*", "/"]
_NUM = re.compile(r"[0-9]+(\.[0-9]+)?([eE][+-]?[0-9]+)?")


@dataclass
class Token:
    kind: str  # keyword ident number string op punct eof
    text: str
    number: float = 0.0
    pos: tuple[int, int] = (0, 0)


def tokenize(text: str) -> list[Token]:
    out: list[Token] = []
    i, line, col = 0, 1, 1
    n = len(text)

    def adv(k: int):
        nonlocal i, line, col
        for _ in range(k):
            if text[i] == "\n":
                line += 1
                col = 1
            else:
                col += 1
            i += 1

    while i < n:
        c = text[i]
        if c in " \t\r\n":
            adv(1)
            continue
        if c == "/" and i + 1 < n and text[i + 1] == "/":
            while i < n and text[i] != "\n":
                adv(1)
            continue
        pos = (line, col)
        if c.isascii() and c.isalpha():
            j = i
            while j < n and text[j].isascii() and (text[j].isalnum() or text[j] == "_"):
                j += 1
            w = text[i:j]
            adv(j - i)
            out.append(Token("keyword" if w in _KEYWORDS else "ident", w, 0.0, pos))
            continue
        if c.isdigit():
            m = _NUM.match(text, i)
            lex = m.group(0)
            adv(len(lex))
            out.append(Token("number", lex, float(lex), pos))
            continue
        if c == '"':
            j = i + 1
            while j < n and text[j] not in '"\n':
                j += 1
            if j >= n or text[j] != '"':
                raise SpecError("lex", "unterminated string literal", pos)
            s = text[i + 1:j]
            adv(j - i + 1)
            out.append(Token("string", s, 0.0, pos))
            continue
        if c in "(),":
            adv(1)
            out.append(Token("punct", c, 0.0, pos))
            continue
        for op in _OPS:
            if text.startswith(op, i):
                adv(len(op))
                out.append(Token("op", op, 0.0, pos))
                break
        else:
            if c == "=":
                adv(1)
                out.append(Token("punct", "=", 0.0, pos))
                continue
            raise SpecError("lex", f"unexpected character '{c}'", pos)
    out.append(Token("eof", "", 0.0, (line, col)))
    return out


# ---------------------------------------------------------------- AST
@dataclass
class Expr:
    kind: str  # num ident apply infix prefix paren
    value: float = 0.0
    name: str = ""
    args: list = field(default_factory=list)
    pos: tuple[int, int] = (0, 0)


@dataclass
class Let:
    name: str
    params: list[str]
    body: Expr
    pos: tuple[int, int]


@dataclass
class Load:
    name: str
    path: str
    pos: tuple[int, int]


@dataclass
class Save:
    path: str
    expr: Expr
    pos: tuple[int, int]


@dataclass
class Print:
    label: str
    expr: Expr
    pos: tuple[int, int]


@dataclass
class Import:
    path: str
    pos: tuple[int, int]


Command = Union[Let, Load, Save, Print, Import]

_PREC = {"|": 1, "&": 2, ">.": 3, ">=.": 3, "<.": 3, "<=.": 3, "=.": 3, "+": 4, "-": 4,
         "*": 5, "/": 5}


class _Parser:
    def __init__(self, toks: list[Token]):
        self.t, self.i = toks, 0

    def peek(self) -> Token:
        return self.t[min(self.i, len(self.t) - 1)]

    def next(self) -> Token:
        tok = self.peek()
        self.i += 1
        return tok

    def err(self, msg: str) -> SpecError:
        return SpecError("parse", msg, self.peek().pos)

    def at(self, kind: str, text: str) -> bool:
        return self.peek().kind == kind and self.peek().text == text

    def expect_punct(self, p: str):
        if not self.at("punct", p):
            raise self.err(f"expected '{p}'")
        self.next()

    def expect_ident(self, what: str) -> str:
        if self.peek().kind != "ident":
            raise self.err(f"expected {what}, got '{self.peek().text}'")
        return self.next().text

    def expect_string(self, what: str) -> str:
        if self.peek().kind != "string":
            raise self.err(f"expected a string for {what}")
        return self.next().text

    def run(self) -> list[Command]:
        prog: list[Command] = []
        declared: set[str] = set()
        while self.peek().kind != "eof":
            t = self.peek()
            if t.kind != "keyword":
                raise self.err(f"expected a command (let, load, save, print, import), got '{t.text}'")
            if t.text == "let":
                d = self.parse_let()
                if d.name in declared:
                    raise SpecError("parse", f"duplicate declaration of '{d.name}'", d.pos)
                declared.add(d.name)
                prog.append(d)
            elif t.text == "load":
                pos = self.next().pos
                name = self.expect_ident("a name after load")
                self.expect_punct("=")
                path = self.expect_string("load path")
                if not path:
                    raise SpecError("parse", "load path must not be empty", pos)
                if name in declared:
                    raise SpecError("parse", f"duplicate declaration of '{name}'", pos)
                declared.add(name)
                prog.append(Load(name, path, pos))
            elif t.text == "save":
                pos = self.next().pos
                path = self.expect_string("save path")
                if not path:
                    raise SpecError("parse", "save path must not be empty", pos)
                prog.append(Save(path, self.parse_expr(), pos))
            elif t.text == "print":
                pos = self.next().pos
                label = self.expect_string("print label")
                prog.append(Print(label, self.parse_expr(), pos))
            else:
                pos = self.next().pos
                path = self.expect_string("import path")
                if not path:
                    raise SpecError("parse", "import path must not be empty", pos)
                prog.append(Import(path, pos))
        return prog

    def parse_let(self) -> Let:
        pos = self.next().pos
        name = self.expect_ident("a name after let")
        params: list[str] = []
        if self.at("punct", "("):
            self.next()
            while True:
                ppos = self.peek().pos
                p = self.expect_ident("a parameter name")
                if p in params:
                    raise SpecError("parse", f"duplicate parameter '{p}'", ppos)
                params.append(p)
                if self.at("punct", ","):
                    self.next()
                    continue
                self.expect_punct(")")
                break
        self.expect_punct("=")
        return Let(name, params, self.parse_expr(), pos)

    def parse_expr(self) -> Expr:
        return self.parse_infix(1)

    def parse_infix(self, level: int) -> Expr:
        if level > 5:
            return self.parse_unary()
        lhs = self.parse_infix(level + 1)
        while self.peek().kind == "op" and _PREC.get(self.peek().text) == level:
            op = self.next()
            rhs = self.parse_infix(level + 1)
            lhs = Expr("infix", name=op.text, args=[lhs, rhs], pos=op.pos)
        return lhs

    def parse_unary(self) -> Expr:
        if self.at("op", "!"):
            op = self.next()
            return Expr("prefix", name="!", args=[self.parse_unary()], pos=op.pos)
        return self.parse_primary()

    def parse_primary(self) -> Expr:
        t = self.peek()
        if t.kind == "number":
            self.next()
            return Expr("num", value=t.number, pos=t.pos)
        if t.kind == "ident":
            name = self.next()
            if self.at("punct", "("):
                self.next()
                args = [self.parse_expr()]
                while self.at("punct", ","):
                    self.next()
                    args.append(self.parse_expr())
                self.expect_punct(")")
                return Expr("apply", name=name.text, args=args, pos=name.pos)
            return Expr("ident", name=name.text, pos=name.pos)
        if t.kind == "punct" and t.text == "(":
            self.next()
            inner = self.parse_expr()
            self.expect_punct(")")
            return Expr("paren", args=[inner], pos=t.pos)
        got = "end of file" if t.kind == "eof" else t.text
        raise self.err(f"expected an expression, got '{got}'")


def parse_text(text: str) -> list[Command]:
    return _Parser(tokenize(text)).run()


# ---------------------------------------------------------------- task graph
@dataclass
class Task:
    opcode: str
    payload: Union[None, float, str]
    deps: tuple[int, ...]


def payload_text(p) -> str:
    """payloadText (task_graph.cpp:18-26): '-', shortest double, or quoted."""
    if p is None:
        return "-"
    if isinstance(p, float):
        if math.isinf(p):
            return "inf" if p > 0 else "-inf"
        if math.isnan(p):
            return "nan"
        s = repr(p)
        if s.endswith(".0"):
            s = s[:-2]
        if "e" in s:
            mant, exp = s.split("e")
            if mant.endswith(".0"):
                mant = mant[:-2]
            sign = "-" if exp.startswith("-") else "+"
            exp = exp.lstrip("+-").lstrip("0") or "0"
            s = f"{mant}e{sign}{exp.zfill(2)}"
        return s
    return f'"{p}"'


class TaskGraph:
    """Hash-consed DAG (task_graph.hpp:30-62); ids are a topological order."""

    def __init__(self):
        self.nodes: list[Task] = []
        self.outputs: list[int] = []
        self._interned: dict = {}

    def intern(self, opcode: str, payload, deps) -> int:
        deps = tuple(deps)
        if isinstance(payload, float):
            pk = ("d", struct.pack("<d", payload))
        elif isinstance(payload, str):
            pk = ("s", payload)
        else:
            pk = ("-",)
        key = (opcode, pk, deps)
        hit = self._interned.get(key)
        if hit is not None:
            return hit
        nid = len(self.nodes)
        assert all(d < nid for d in deps)
        self.nodes.append(Task(opcode, payload, deps))
        self._interned[key] = nid
        return nid

    def add_output(self, nid: int) -> None:
        if nid not in self.outputs:
            self.outputs.append(nid)

    def node_count(self) -> int:
        return len(self.nodes)

    def toposort(self) -> list[int]:
        return list(range(len(self.nodes)))

    def count_opcode(self, op: str) -> int:
        return sum(1 for t in self.nodes if t.opcode == op)

    def dump(self) -> str:
        lines = []
        for i, t in enumerate(self.nodes):
            deps = ",".join(str(d) for d in t.deps) if t.deps else "-"
            lines.append(f"{i} {t.opcode} {payload_text(t.payload)} {deps}")
        return "".join(l + "\n" for l in lines)


BUILTINS = {"near": 1, "reach": 2, "intensity": 1, "volume": 1, "!": 1, "&": 2, "|": 2, "+": 2,
            "-": 2, "*": 2, "/": 2, ">.": 2, ">=.": 2, "<.": 2, "<=.": 2, "=.": 2,
            "maxvol": 1, "components": 1}

Resolver = Callable[[str], str]


def default_resolver(path: str) -> str:
    if path in ("stdlib", "<builtin-stdlib>"):
        return STDLIB
    with open(path) as f:
        return f.read()


class _Expander:
    def __init__(self, resolver: Optional[Resolver]):
        self.g = TaskGraph()
        self.resolver = resolver
        self.globals: dict = {}
        self.imported: set[str] = set()

    def process(self, prog: list[Command]):
        for c in prog:
            if isinstance(c, Let):
                self.check_expr(c.body, c.name, set(c.params))
                self.declare(c.name, c.pos, ("macro", c.params, c.body))
            elif isinstance(c, Load):
                self.declare(c.name, c.pos, ("load", c.path))
            elif isinstance(c, Save):
                self.g.add_output(self.g.intern("save", c.path, [self.expr(c.expr, None)]))
            elif isinstance(c, Print):
                self.g.add_output(self.g.intern("print", c.label, [self.expr(c.expr, None)]))
            else:
                if self.resolver is None:
                    raise SpecError("expand", "import is not available here", c.pos)
                if c.path in self.imported:
                    continue
                self.imported.add(c.path)
                try:
                    text = self.resolver(c.path)
                except OSError:
                    raise SpecError("expand", f"cannot open import file: {c.path}") from None
                self.process(parse_text(text))

    def declare(self, name, pos, g):
        if name in BUILTINS:
            raise SpecError("expand", f"'{name}' redefines a built-in", pos)
        if name in self.globals:
            raise SpecError("expand", f"duplicate top-level name '{name}' across files", pos)
        self.globals[name] = g

    def check_expr(self, e: Expr, me: str, params: set):
        k = e.kind
        if k == "ident":
            if e.name in params:
                return
            if e.name == me:
                raise SpecError("expand", f"'{e.name}' used inside its own definition (lets are "
                                          "non-recursive)", e.pos)
            g = self.globals.get(e.name)
            if g is None:
                raise SpecError("expand", f"unbound identifier '{e.name}'", e.pos)
            if g[0] == "macro" and g[1]:
                raise SpecError("expand", f"'{e.name}' takes {len(g[1])} argument(s) but is used "
                                          "without any", e.pos)
        elif k == "apply":
            self.check_call(e.name, len(e.args), me, params, e.pos)
            for a in e.args:
                self.check_expr(a, me, params)
        elif k in ("infix", "prefix", "paren"):
            for a in e.args:
                self.check_expr(a, me, params)

    def check_call(self, fn, argc, me, params, pos):
        if fn in params:
            raise SpecError("expand", f"parameter '{fn}' cannot be applied as a function", pos)
        if fn == me:
            raise SpecError("expand", f"'{fn}' used inside its own definition (lets are "
                                      "non-recursive)", pos)
        if fn in BUILTINS:
            if BUILTINS[fn] != argc:
                raise SpecError("expand", f"'{fn}' expects {BUILTINS[fn]} argument(s), got {argc}",
                                pos)
            return
        g = self.globals.get(fn)
        if g is None:
            raise SpecError("expand", f"unbound identifier '{fn}'", pos)
        if g[0] != "macro":
            raise SpecError("expand", f"'{fn}' is an image, not a function", pos)
        if len(g[1]) != argc:
            raise SpecError("expand", f"'{fn}' expects {len(g[1])} argument(s), got {argc}", pos)

    def expr(self, e: Expr, params: Optional[dict]) -> int:
        k = e.kind
        if k == "num":
            return self.g.intern("const", float(e.value), [])
        if k == "ident":
            if params and e.name in params:
                return params[e.name]
            g = self.globals.get(e.name)
            if g is None:
                raise SpecError("expand", f"unbound identifier '{e.name}'", e.pos)
            if g[0] == "load":
                return self.g.intern("load", g[1], [])
            if g[1]:
                raise SpecError("expand", f"'{e.name}' takes {len(g[1])} argument(s) but is used "
                                          "without any", e.pos)
            return self.expr(g[2], None)
        if k == "apply":
            return self.call(e, params)
        if k == "infix":
            l = self.expr(e.args[0], params)
            r = self.expr(e.args[1], params)
            return self.g.intern(e.name, None, [l, r])
        if k == "prefix":
            return self.g.intern(e.name, None, [self.expr(e.args[0], params)])
        return self.expr(e.args[0], params)

    def call(self, e: Expr, params: Optional[dict]) -> int:
        fn = e.name
        if params and fn in params:
            raise SpecError("expand", f"parameter '{fn}' cannot be applied as a function", e.pos)
        if fn in BUILTINS:
            if BUILTINS[fn] != len(e.args):
                raise SpecError("expand", f"'{fn}' expects {BUILTINS[fn]} argument(s), got "
                                          f"{len(e.args)}", e.pos)
            deps = [self.expr(a, params) for a in e.args]
            return self.g.intern(fn, None, deps)
        g = self.globals.get(fn)
        if g is None:
            raise SpecError("expand", f"unbound identifier '{fn}'", e.pos)
        if g[0] != "macro":
            raise SpecError("expand", f"'{fn}' is an image, not a function", e.pos)
        if len(g[1]) != len(e.args):
            raise SpecError("expand", f"'{fn}' expects {len(g[1])} argument(s), got "
                                      f"{len(e.args)}", e.pos)
        env = {}
        for p, a in zip(g[1], e.args):
            env[p] = self.expr(a, params)
        return self.expr(g[2], env)


def expand(prog: list[Command], resolver: Optional[Resolver] = default_resolver) -> TaskGraph:
    ex = _Expander(resolver)
    ex.process(prog)
    return ex.g


def _deep(fn, *a):
    """Runs a recursive-descent pass on a thread with a large stack: 1000-deep
    formulas (BASELINE config 2) nest a few thousand Python frames."""
    import sys
    import threading
    out: dict = {}

    def body():
        try:
            out["v"] = fn(*a)
        except BaseException as e:  # re-raised on the caller's thread
            out["e"] = e

    old_limit = sys.getrecursionlimit()
    old_stack = threading.stack_size()
    sys.setrecursionlimit(max(old_limit, 200000))
    threading.stack_size(512 << 20)
    try:
        t = threading.Thread(target=body)
        t.start()
        t.join()
    finally:
        threading.stack_size(old_stack)
        sys.setrecursionlimit(old_limit)
    if "e" in out:
        raise out["e"]
    return out["v"]


def compile_text(text: str, with_stdlib: bool = True,
                 resolver: Optional[Resolver] = default_resolver) -> TaskGraph:
    """parse + stdlib import + expand, the runSpec sequence (cli.cpp:62-75)."""
    if with_stdlib:
        text = 'import "stdlib"\n' + text
    return _deep(lambda: expand(parse_text(text), resolver))
