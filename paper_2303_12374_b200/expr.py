"""Restriction / launch-geometry expression language.

Semantics follow the reference grammar (pkg/src/kltune/expr.py:1-19) exactly:
C precedence ``|| < && < comparisons < + - < * / % < unary (- !)``, all binary
levels left-associative, 64-bit checked integer arithmetic with truncating
``/`` and ``%`` (expr.py:351-353, 444-447), ``ceil_div(a, b)`` defined only for
``a >= 0, b > 0`` (expr.py:394-399), short-circuit ``&&``/``||`` (expr.py:409-415)
and strings comparable only with ``==``/``!=`` (expr.py:420-430).

Implementation differs from the reference: the parser is a precedence-climbing
loop over one operator table, and every tree can be lowered once to a Python
closure (``compile_expr``) so the runtime dispatch path evaluates launch
geometry without re-walking the tree.  ``evaluate`` is defined as "compile and
call", so both entry points share one set of semantics and error messages.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterator, Mapping, Union

__all__ = [
    "Value", "Env", "Expr", "IntLit", "BoolLit", "StrLit", "Ident", "Unary", "Binary",
    "Call", "ParseError", "EvalError", "FUNCTIONS", "I64_MIN", "I64_MAX", "parse",
    "to_text", "evaluate", "evaluate_bool", "evaluate_int", "identifiers", "compile_expr",
]

Value = Union[int, bool, str]
Env = Mapping[str, Value]

I64_MIN = -(1 << 63)
I64_MAX = (1 << 63) - 1

#: callable name -> arity
FUNCTIONS = {"ceil_div": 2, "min": 2, "max": 2}


class ParseError(Exception):
    """Malformed expression text; ``offset`` indexes the offending character."""

    def __init__(self, message: str, offset: int) -> None:
        super().__init__(f"{message} (at offset {offset})")
        self.offset = offset


class EvalError(Exception):
    """Type error, unbound name, domain error or 64-bit overflow."""


# ---------------------------------------------------------------------------
# Tree nodes (value objects; structural equality is what round-trips test)


@dataclass(frozen=True)
class IntLit:
    value: int


@dataclass(frozen=True)
class BoolLit:
    value: bool


@dataclass(frozen=True)
class StrLit:
    value: str


@dataclass(frozen=True)
class Ident:
    name: str


@dataclass(frozen=True)
class Unary:
    op: str
    operand: "Expr"


@dataclass(frozen=True)
class Binary:
    op: str
    left: "Expr"
    right: "Expr"


@dataclass(frozen=True)
class Call:
    name: str
    args: tuple["Expr", ...]


Expr = Union[IntLit, BoolLit, StrLit, Ident, Unary, Binary, Call]

# Binding power of every binary operator; higher binds tighter.
_BINARY_POWER = {
    "||": 1,
    "&&": 2,
    "==": 3, "!=": 3, "<": 3, "<=": 3, ">": 3, ">=": 3,
    "+": 4, "-": 4,
    "*": 5, "/": 5, "%": 5,
}
_PREFIX_POWER = 6
_PUNCT2 = frozenset(("==", "!=", "<=", ">=", "&&", "||"))
_PUNCT1 = frozenset("+-*/%<>!(),")


# ---------------------------------------------------------------------------
# Lexer


@dataclass(frozen=True)
class _Tok:
    kind: str  # num | name | text | punct | end
    text: str
    pos: int


def _lex(src: str) -> Iterator[_Tok]:
    pos, end = 0, len(src)
    while pos < end:
        ch = src[pos]
        if ch.isspace():
            pos += 1
        elif ch.isdigit():
            stop = pos + 1
            while stop < end and src[stop].isdigit():
                stop += 1
            yield _Tok("num", src[pos:stop], pos)
            pos = stop
        elif ch == "_" or ch.isalpha():
            stop = pos + 1
            while stop < end and (src[stop] == "_" or src[stop].isalnum()):
                stop += 1
            yield _Tok("name", src[pos:stop], pos)
            pos = stop
        elif ch == '"':
            start, pos, chars = pos, pos + 1, []
            while True:
                if pos >= end:
                    raise ParseError("unterminated string literal", start)
                ch = src[pos]
                if ch == '"':
                    pos += 1
                    break
                if ch == "\\":
                    if pos + 1 >= end:
                        raise ParseError("unterminated string escape", pos)
                    nxt = src[pos + 1]
                    if nxt != '"' and nxt != "\\":
                        raise ParseError(f"unsupported escape '\\{nxt}'", pos)
                    chars.append(nxt)
                    pos += 2
                else:
                    chars.append(ch)
                    pos += 1
            yield _Tok("text", "".join(chars), start)
        elif src[pos:pos + 2] in _PUNCT2:
            yield _Tok("punct", src[pos:pos + 2], pos)
            pos += 2
        elif ch in _PUNCT1:
            yield _Tok("punct", ch, pos)
            pos += 1
        else:
            raise ParseError(f"unexpected character {ch!r}", pos)
    yield _Tok("end", "", end)


# ---------------------------------------------------------------------------
# Parser: precedence climbing


class _Reader:
    __slots__ = ("toks", "i")

    def __init__(self, src: str) -> None:
        self.toks = list(_lex(src))
        self.i = 0

    def peek(self) -> _Tok:
        return self.toks[self.i]

    def take(self) -> _Tok:
        tok = self.toks[self.i]
        self.i += 1
        return tok

    def is_punct(self, text: str) -> bool:
        tok = self.toks[self.i]
        return tok.kind == "punct" and tok.text == text

    def expect(self, text: str) -> None:
        if not self.is_punct(text):
            raise ParseError(f"expected '{text}'", self.peek().pos)
        self.i += 1

    def binary(self, floor: int) -> Expr:
        lhs = self.prefix()
        while True:
            tok = self.peek()
            power = _BINARY_POWER.get(tok.text) if tok.kind == "punct" else None
            if power is None or power < floor:
                return lhs
            self.i += 1
            lhs = Binary(tok.text, lhs, self.binary(power + 1))

    def prefix(self) -> Expr:
        tok = self.peek()
        if tok.kind == "punct" and tok.text in ("-", "!"):
            self.i += 1
            return Unary(tok.text, self.prefix())
        return self.atom()

    def atom(self) -> Expr:
        tok = self.take()
        if tok.kind == "num":
            number = int(tok.text)
            if number > I64_MAX:
                raise ParseError("integer literal out of 64-bit range", tok.pos)
            return IntLit(number)
        if tok.kind == "text":
            return StrLit(tok.text)
        if tok.kind == "name":
            if tok.text in ("true", "false"):
                return BoolLit(tok.text == "true")
            if not self.is_punct("("):
                return Ident(tok.text)
            arity = FUNCTIONS.get(tok.text)
            if arity is None:
                raise ParseError(f"unknown function '{tok.text}'", tok.pos)
            self.i += 1
            args = [self.binary(1)]
            while self.is_punct(","):
                self.i += 1
                args.append(self.binary(1))
            self.expect(")")
            if len(args) != arity:
                raise ParseError(
                    f"'{tok.text}' takes {arity} arguments, got {len(args)}", tok.pos
                )
            return Call(tok.text, tuple(args))
        if tok.kind == "punct" and tok.text == "(":
            inner = self.binary(1)
            self.expect(")")
            return inner
        self.i -= 1
        if tok.kind == "end":
            raise ParseError("unexpected end of input", tok.pos)
        raise ParseError(f"unexpected token {tok.text!r}", tok.pos)


def parse(text: str) -> Expr:
    """Parse expression text into a tree."""
    reader = _Reader(text)
    tree = reader.binary(1)
    tail = reader.peek()
    if tail.kind != "end":
        raise ParseError(f"unexpected trailing input {tail.text!r}", tail.pos)
    return tree


# ---------------------------------------------------------------------------
# Printer (minimal parentheses; parse(to_text(e)) == e)


def to_text(expr: Expr) -> str:
    return _render(expr, 0)


def _render(node: Expr, context: int) -> str:
    kind = type(node)
    if kind is IntLit:
        return str(node.value)
    if kind is BoolLit:
        return "true" if node.value else "false"
    if kind is StrLit:
        escaped = node.value.replace("\\", "\\\\").replace('"', '\\"')
        return '"' + escaped + '"'
    if kind is Ident:
        return node.name
    if kind is Call:
        return node.name + "(" + ", ".join(_render(a, 0) for a in node.args) + ")"
    if kind is Unary:
        body = _render(node.operand, _PREFIX_POWER)
        gap = " " if node.op == "-" and body[:1] == "-" else ""
        text = node.op + gap + body
        return "(" + text + ")" if context > _PREFIX_POWER else text
    if kind is Binary:
        power = _BINARY_POWER[node.op]
        text = f"{_render(node.left, power)} {node.op} {_render(node.right, power + 1)}"
        return "(" + text + ")" if power < context else text
    raise TypeError(f"not an expression node: {node!r}")


# ---------------------------------------------------------------------------
# Evaluation: lower to closures once, call many times

Thunk = Callable[[Env], Value]


def _is_int(v: object) -> bool:
    return type(v) is int or (isinstance(v, int) and not isinstance(v, bool))


def _want_int(v: Value, what: str) -> int:
    if not _is_int(v):
        raise EvalError(f"'{what}' requires integer operands, got {type(v).__name__}")
    return v


def _want_bool(v: Value, what: str) -> bool:
    if not isinstance(v, bool):
        raise EvalError(f"'{what}' requires boolean operands, got {type(v).__name__}")
    return v


def _in_range(v: int, what: str) -> int:
    if v < I64_MIN or v > I64_MAX:
        raise EvalError(f"64-bit overflow in {what}")
    return v


def _tdiv(a: int, b: int) -> int:
    """C-style quotient (rounds toward zero)."""
    q = abs(a) // abs(b)
    return -q if (a < 0) != (b < 0) else q


def _arith_add(a, b):
    return _in_range(a + b, "addition")


def _arith_sub(a, b):
    return _in_range(a - b, "subtraction")


def _arith_mul(a, b):
    return _in_range(a * b, "multiplication")


def _arith_div(a, b):
    if b == 0:
        raise EvalError("division by zero")
    return _in_range(_tdiv(a, b), "division")


def _arith_mod(a, b):
    if b == 0:
        raise EvalError("modulo by zero")
    return a - _tdiv(a, b) * b


_INT_OPS = {
    "+": _arith_add,
    "-": _arith_sub,
    "*": _arith_mul,
    "/": _arith_div,
    "%": _arith_mod,
    "<": lambda a, b: a < b,
    "<=": lambda a, b: a <= b,
    ">": lambda a, b: a > b,
    ">=": lambda a, b: a >= b,
}


def _fn_ceil_div(a: int, b: int) -> int:
    if a < 0 or b <= 0:
        raise EvalError(f"ceil_div requires a >= 0 and b > 0, got ({a}, {b})")
    return _in_range(-(-a // b), "ceil_div")


_FUNCS = {"ceil_div": _fn_ceil_div, "min": min, "max": max}


def _lower(node: Expr) -> Thunk:
    kind = type(node)
    if kind in (IntLit, BoolLit, StrLit):
        const = node.value
        return lambda env: const
    if kind is Ident:
        name = node.name

        def lookup(env: Env) -> Value:
            try:
                return env[name]
            except KeyError:
                raise EvalError(f"unbound identifier '{name}'") from None

        return lookup
    if kind is Unary:
        inner = _lower(node.operand)
        if node.op == "!":
            return lambda env: not _want_bool(inner(env), "!")
        return lambda env: _in_range(-_want_int(inner(env), "unary -"), "negation")
    if kind is Call:
        fn = _FUNCS.get(node.name)
        thunks = [_lower(a) for a in node.args]
        label = node.name

        def call(env: Env) -> Value:
            values = [t(env) for t in thunks]
            ints = [_want_int(v, label) for v in values]
            if fn is None:
                raise EvalError(f"unknown function '{label}'")
            return fn(*ints)

        return call
    if kind is Binary:
        op = node.op
        left, right = _lower(node.left), _lower(node.right)
        if op == "&&":
            return lambda env: _want_bool(left(env), op) and _want_bool(right(env), op)
        if op == "||":
            return lambda env: _want_bool(left(env), op) or _want_bool(right(env), op)
        if op in ("==", "!="):
            negate = op == "!="

            def equality(env: Env) -> bool:
                a, b = left(env), right(env)
                if not ((_is_int(a) and _is_int(b)) or (type(a) is str and type(b) is str)):
                    raise EvalError(
                        f"'{op}' requires two integers or two strings, got "
                        f"{type(a).__name__} and {type(b).__name__}"
                    )
                return (a != b) if negate else (a == b)

            return equality
        impl = _INT_OPS.get(op)
        if impl is None:
            raise EvalError(f"unknown operator '{op}'")

        def arith(env: Env) -> Value:
            a, b = left(env), right(env)
            return impl(_want_int(a, op), _want_int(b, op))

        return arith
    raise TypeError(f"not an expression node: {node!r}")


_LOWERED: dict[int, tuple[Expr, Thunk]] = {}


def compile_expr(expr: Expr) -> Thunk:
    """Closure evaluating ``expr``; cached per tree object."""
    hit = _LOWERED.get(id(expr))
    if hit is not None and hit[0] is expr:
        return hit[1]
    thunk = _lower(expr)
    if len(_LOWERED) > 65536:
        _LOWERED.clear()
    _LOWERED[id(expr)] = (expr, thunk)
    return thunk


def evaluate(expr: Expr, env: Env) -> Value:
    """Value of ``expr`` under ``env`` (pure; unbound names are errors)."""
    return compile_expr(expr)(env)


def evaluate_bool(expr: Expr, env: Env) -> bool:
    result = evaluate(expr, env)
    if not isinstance(result, bool):
        raise EvalError(f"expression is not boolean-typed (got {type(result).__name__})")
    return result


def evaluate_int(expr: Expr, env: Env) -> int:
    result = evaluate(expr, env)
    if not _is_int(result):
        raise EvalError(f"expression is not integer-typed (got {type(result).__name__})")
    return result


def identifiers(expr: Expr) -> set[str]:
    """Every identifier name in the tree."""
    found: set[str] = set()
    stack = [expr]
    while stack:
        node = stack.pop()
        kind = type(node)
        if kind is Ident:
            found.add(node.name)
        elif kind is Unary:
            stack.append(node.operand)
        elif kind is Binary:
            stack.append(node.left)
            stack.append(node.right)
        elif kind is Call:
            stack.extend(node.args)
    return found
