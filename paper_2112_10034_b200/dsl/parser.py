"""Lexer + parser for `.spk` kernels (reference grammar: docs/grammar.md;
reference entry point: dsl/parser.py:351 ``parse_module``).

Written independently of the reference: a table-driven tokenizer and a
precedence-climbing expression parser.  It accepts everything the reference
grammar accepts and produces the same exception classes (ParseError with
``line:col``, SemanticError, UnsupportedFeatureError).  Extensions (native
on B200): ``shfl_up``, ``shfl_xor``, ``shfl_idx``, ``ballot``, ``reduce_add``,
non-literal masks, CUDA spellings (``__shfl_down_sync(m, v, d)``,
``__shfl_up_sync``, ``__shfl_xor_sync``, ``__shfl_sync``, ``__ballot_sync``,
``__all_sync``, ``__any_sync``, ``__reduce_add_sync``) and
``extern shared <kind> name[];`` (dynamic shared memory).
"""

from __future__ import annotations

import re
from dataclasses import dataclass

from ..errors import ParseError, SemanticError, UnsupportedFeatureError
from . import nodes as n

KEYWORDS = {"__global__", "void", "if", "else", "for", "return", "i32", "f32", "global",
            "shared", "extern", "__syncthreads", "__syncwarp"}

REJECTED = {
    "grid_sync": "grid-level synchronization is unsupported (no grid-wide barrier)",
    "this_grid": "grid-level cooperative groups are unsupported",
    "coalesced_threads": "dynamic (activated-thread) groups are unsupported",
    "switch": "switch statements are not part of this language",
    "goto": "goto is not part of this language",
}

# collective spelling -> (op, number of value args, has leading mask)
CALLS = {
    "shfl_down": ("shfl_down", 2, None), "shfl_up": ("shfl_up", 2, None),
    "shfl_xor": ("shfl_xor", 2, None), "shfl_idx": ("shfl_idx", 2, None),
    "vote_all": ("vote_all", 1, None), "vote_any": ("vote_any", 1, None),
    "ballot": ("ballot", 1, None), "reduce_add": ("reduce_add", 1, None),
    "__shfl_down_sync": ("shfl_down", 2, True), "__shfl_up_sync": ("shfl_up", 2, True),
    "__shfl_xor_sync": ("shfl_xor", 2, True), "__shfl_sync": ("shfl_idx", 2, True),
    "__all_sync": ("vote_all", 1, True), "__any_sync": ("vote_any", 1, True),
    "__ballot_sync": ("ballot", 1, True), "__reduce_add_sync": ("reduce_add", 1, True),
}

_TOKEN_RE = re.compile(r"""
    (?P<ws>[ \t\r]+) | (?P<nl>\n) | (?P<lc>//[^\n]*) | (?P<bc>/\*.*?\*/) |
    (?P<float>(\d+\.\d*|\.\d+)([eE][+-]?\d+)?f?|\d+[eE][+-]?\d+f?) |
    (?P<int>0[xX][0-9a-fA-F]+|\d+) |
    (?P<builtin>(threadIdx|blockIdx|blockDim|gridDim)\.x\b) |
    (?P<ident>[A-Za-z_][A-Za-z_0-9]*) |
    (?P<punct><<|>>|==|!=|<=|>=|&&|\|\||\+=|-=|\*=|/=|%=|\+\+|--|[(){}\[\];,=<>+\-*/%!&|^~])
""", re.X | re.S)


@dataclass(frozen=True)
class Tok:
    kind: str  # ident | keyword | builtin | int | float | punct | eof
    text: str
    line: int
    col: int


def tokenize(src: str) -> list[Tok]:
    out, pos, line, col = [], 0, 1, 1
    while pos < len(src):
        m = _TOKEN_RE.match(src, pos)
        if not m:
            raise ParseError(f"unexpected character {src[pos]!r}", line, col)
        kind, text = m.lastgroup, m.group()
        if kind in ("ws", "lc"):
            pass
        elif kind == "nl":
            line, col = line + 1, 0
        elif kind == "bc":
            nls = text.count("\n")
            if nls:
                line += nls
                col = len(text) - text.rfind("\n") - 1
        else:
            if kind == "ident" and text in KEYWORDS:
                kind = "keyword"
            out.append(Tok(kind, text, line, col))
        col += len(text) if kind != "nl" else 1
        pos = m.end()
    out.append(Tok("eof", "", line, col))
    return out


# binary precedence (higher binds tighter); all left-associative
_PREC = {"||": 1, "&&": 2, "==": 3, "!=": 3, "<": 3, "<=": 3, ">": 3, ">=": 3,
         "+": 4, "-": 4, "*": 5, "/": 5, "%": 5}
_ASSIGN = {"=": None, "+=": "+", "-=": "-", "*=": "*", "/=": "/", "%=": "%"}
_UNSUPPORTED_OPS = {"<<": "shift", ">>": "shift", "&": "bitwise and", "|": "bitwise or",
                    "^": "bitwise xor", "~": "bitwise not"}


def _wrap32(v: int) -> int:
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= 1 << 31 else v


class _Parser:
    def __init__(self, toks: list[Tok]):
        self.toks, self.i = toks, 0

    # -- token helpers
    def peek(self, k: int = 0) -> Tok:
        return self.toks[min(self.i + k, len(self.toks) - 1)]

    def take(self) -> Tok:
        t = self.peek()
        self.i += 1
        return t

    def at(self, text: str) -> bool:
        return self.peek().text == text and self.peek().kind != "eof"

    def eat(self, text: str) -> bool:
        if self.at(text):
            self.i += 1
            return True
        return False

    def need(self, text: str) -> Tok:
        t = self.peek()
        if t.text != text or t.kind == "eof":
            self.error(f"expected {text!r}, found {t.text or 'end of input'!r}")
        return self.take()

    def error(self, msg: str, tok: Tok | None = None):
        t = tok or self.peek()
        raise ParseError(msg, t.line, t.col)

    def unsupported(self, msg: str, tok: Tok):
        raise UnsupportedFeatureError(f"{tok.line}:{tok.col}: unsupported feature: {msg}")

    # -- module / kernel
    def module(self) -> n.KernelModule:
        mod = n.KernelModule()
        while self.peek().kind != "eof":
            mod.kernels.append(self.kernel())
        if not mod.kernels:
            self.error("no kernel in module")
        return mod

    def kernel(self) -> n.KernelDef:
        self.need("__global__")
        self.need("void")
        name = self.ident()
        self.need("(")
        params = []
        if not self.at(")"):
            params.append(self.param())
            while self.eat(","):
                params.append(self.param())
        self.need(")")
        return n.KernelDef(name, tuple(params), self.block())

    def param(self) -> n.Param:
        if self.eat("global"):
            kind = self.kind()
            self.need("*")
            return n.Param(self.ident(), kind, True)
        kind = self.kind()
        return n.Param(self.ident(), kind, False)

    def kind(self) -> str:
        t = self.peek()
        if t.text in ("i32", "f32"):
            return self.take().text
        if t.kind == "ident" and t.text in ("u8", "u32", "i64", "f64", "int", "float"):
            self.unsupported(f"type {t.text!r} (the language has i32 and f32)", t)
        self.error(f"expected a type (i32 or f32), found {t.text!r}")

    def ident(self) -> str:
        t = self.peek()
        if t.kind != "ident":
            self.error(f"expected an identifier, found {t.text or 'end of input'!r}")
        return self.take().text

    # -- statements
    def block(self) -> tuple:
        self.need("{")
        body = []
        while not self.at("}"):
            if self.peek().kind == "eof":
                self.error("unterminated block")
            body.append(self.stmt())
        self.need("}")
        return tuple(body)

    def body(self) -> tuple:
        return self.block() if self.at("{") else (self.stmt(),)

    def stmt(self):
        t = self.peek()
        if t.text in REJECTED and t.kind == "ident":
            self.unsupported(REJECTED[t.text], t)
        if t.text in ("shared", "extern"):
            return self.decl_shared()
        if t.text in ("i32", "f32"):
            s = self.decl_local()
            self.need(";")
            return s
        if t.text == "if":
            self.take()
            self.need("(")
            cond = self.expr()
            self.need(")")
            then = self.body()
            orelse = self.body() if self.eat("else") else None
            return n.If(cond, then, orelse)
        if t.text == "for":
            return self.for_stmt()
        if t.text == "__syncthreads":
            self.take()
            self.need("(")
            self.need(")")
            self.need(";")
            return n.SyncThreads()
        if t.text == "__syncwarp":
            self.take()
            self.need("(")
            mask = None if self.at(")") else self.expr()
            self.need(")")
            self.need(";")
            return n.SyncWarp(_full_mask_as_none(mask))
        if t.text == "return":
            self.take()
            self.need(";")
            return n.Return()
        s = self.assign()
        self.need(";")
        return s

    def decl_local(self) -> n.DeclLocal:
        kind = self.kind()
        name = self.ident()
        init = self.expr() if self.eat("=") else None
        return n.DeclLocal(kind, name, init)

    def decl_shared(self) -> n.DeclShared:
        dynamic = self.eat("extern")
        self.need("shared")
        kind = self.kind()
        name = self.ident()
        self.need("[")
        length = None
        if not dynamic:
            t = self.peek()
            if t.kind != "int":
                self.error("shared array length must be a compile-time integer constant")
            length = int(self.take().text, 0)
            if length <= 0:
                raise SemanticError(f"shared array {name!r} must have positive length",
                                    t.line, t.col)
        self.need("]")
        self.need(";")
        return n.DeclShared(kind, name, length)

    def for_stmt(self) -> n.For:
        self.need("for")
        self.need("(")
        if self.peek().text in ("i32", "f32"):
            init = self.decl_local()
            if init.init is None:
                self.error("for-loop declaration needs an initializer")
        else:
            init = self.assign()
        self.need(";")
        cond = self.expr()
        self.need(";")
        step = self.assign(allow_incdec=True)
        self.need(")")
        return n.For(init, cond, step, self.body())

    def assign(self, allow_incdec: bool = False) -> n.Assign:
        t0 = self.peek()
        name = self.ident()
        if self.eat("["):
            idx = self.expr()
            self.need("]")
            target, ref = n.IndexTarget(name, idx), n.IndexExpr(name, idx)
        else:
            target, ref = n.VarTarget(name), n.VarRef(name)
        op = self.peek()
        if op.text in ("++", "--"):
            if not allow_incdec:
                self.error(f"{op.text!r} is only allowed as a for-loop step", op)
            self.take()
            return n.Assign(target, n.Binary("+" if op.text == "++" else "-", ref, n.IntLit(1)))
        if op.text not in _ASSIGN:
            if op.text == "(":
                if name in REJECTED:
                    self.unsupported(REJECTED[name], t0)
                self.error(f"unknown function {name!r}", t0)
            self.error(f"expected an assignment operator, found {op.text!r}", op)
        self.take()
        value = self.expr()
        base = _ASSIGN[op.text]
        return n.Assign(target, value if base is None else n.Binary(base, ref, value))

    # -- expressions (precedence climbing)
    def expr(self, min_prec: int = 1):
        left = self.unary()
        while True:
            t = self.peek()
            if t.kind == "punct" and t.text in _UNSUPPORTED_OPS:
                self.unsupported(f"{_UNSUPPORTED_OPS[t.text]} operator {t.text!r}", t)
            prec = _PREC.get(t.text) if t.kind == "punct" else None
            if prec is None or prec < min_prec:
                return left
            self.take()
            left = n.Binary(t.text, left, self.expr(prec + 1))

    def unary(self):
        t = self.peek()
        if t.kind == "punct" and t.text in ("-", "!"):
            self.take()
            operand = self.unary()
            if t.text == "-" and isinstance(operand, n.IntLit):
                return n.IntLit(_wrap32(-operand.value))  # fold "-1" (masks, constants)
            return n.Unary(t.text, operand)
        if t.kind == "punct" and t.text in _UNSUPPORTED_OPS:
            self.unsupported(f"{_UNSUPPORTED_OPS[t.text]} operator {t.text!r}", t)
        return self.primary()

    def primary(self):
        t = self.peek()
        if t.kind == "int":
            self.take()
            return n.IntLit(_wrap32(int(t.text, 0)))
        if t.kind == "float":
            self.take()
            return n.FloatLit(float(t.text.rstrip("fF")))
        if t.kind == "builtin":
            self.take()
            return n.BuiltinRef(t.text)
        if self.eat("("):
            e = self.expr()
            self.need(")")
            return e
        if t.kind != "ident":
            self.error(f"expected an expression, found {t.text or 'end of input'!r}")
        if t.text in REJECTED:
            self.unsupported(REJECTED[t.text], t)
        if t.text in CALLS and self.peek(1).text == "(":
            return self.call()
        name = self.take().text
        if self.at("("):
            self.error(f"unknown function {name!r}", t)
        if self.eat("["):
            idx = self.expr()
            self.need("]")
            return n.IndexExpr(name, idx)
        return n.VarRef(name)

    def call(self) -> n.CollectiveCall:
        t = self.take()
        op, nargs, mask_first = CALLS[t.text]
        self.need("(")
        args = [self.expr()]
        while self.eat(","):
            args.append(self.expr())
        self.need(")")
        mask = None
        if mask_first or len(args) == nargs + 1:
            if len(args) != nargs + 1:
                raise ParseError(f"{t.text} expects a mask and {nargs} argument(s)", t.line, t.col)
            mask, args = args[0], args[1:]
        if len(args) != nargs:
            raise ParseError(f"{t.text} expects {nargs} argument(s)", t.line, t.col)
        return n.CollectiveCall(op, tuple(args), _full_mask_as_none(mask))


def _full_mask_as_none(mask):
    if isinstance(mask, n.IntLit) and (mask.value & 0xFFFFFFFF) == n.FULL_MASK:
        return None  # the reference's only mask: all lanes
    return mask


def parse_module(source: str) -> n.KernelModule:
    """Parse and check a module (reference dsl/parser.py:351-357)."""
    module = _Parser(tokenize(source)).module()
    from .checker import check_kernel
    for k in module.kernels:
        check_kernel(k)
    return module
