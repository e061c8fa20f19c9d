"""Source construction for generated kernels: placeholders, a tiny template
language, and a C/CUDA syntax tree with a deterministic printer.

Mirrors the substrate of the reference (``src/csyntax.py:73-236`` for
``substitute``/``render``, ``:242-530`` for the tree and ``emit``) with the
same observable behaviour, so generated text is byte-stable and safe to hash
into cache keys.  The B200 kernel templates under ``templates/`` are
expanded with :func:`render`.

* ``substitute(text, bindings)`` replaces ``${name}`` markers only.
* ``render(text, context)`` adds ``{% for v in a..b %}`` (half-open range)
  and ``{% if cond %}`` blocks, then substitutes.
* ``emit(node)`` prints a tree of :class:`CNode` values (4-space indent).
"""

from __future__ import annotations

import re
from dataclasses import dataclass

__all__ = [
    "TemplateError", "MalformedPlaceholder", "UnboundPlaceholder",
    "UnboundVariable", "NonIntegerBound", "UnclosedBlock", "IllFormedTree",
    "substitute", "render", "CType", "CNode", "Raw", "Lit", "Ident", "Index",
    "BinOp", "Call", "Assign", "Decl", "Block", "For", "If", "Param",
    "FunctionDef", "TranslationUnit", "counted_for", "emit",
    "unrolled_add_template", "unrolled_add_ast", "UNROLLED_ADD_TEMPLATE",
]


class TemplateError(Exception):
    """Base class of text-template failures."""


class MalformedPlaceholder(TemplateError):
    """``${`` without a closing brace, or a body that is not an identifier."""


class UnboundPlaceholder(TemplateError):
    def __init__(self, name: str) -> None:
        super().__init__(f"placeholder ${{{name}}} has no binding")
        self.name = name


class UnboundVariable(TemplateError):
    def __init__(self, name: str) -> None:
        super().__init__(f"template variable {name!r} is not defined")
        self.name = name


class NonIntegerBound(TemplateError):
    """A ``for`` bound resolved to something other than an int."""


class UnclosedBlock(TemplateError):
    """Unterminated or mismatched ``{% ... %}`` block."""


class IllFormedTree(Exception):
    """A node sits where its kind is not allowed; ``path`` locates it."""

    def __init__(self, path: str, reason: str) -> None:
        super().__init__(f"{path}: {reason}")
        self.path = path
        self.reason = reason


# --- ${name} substitution --------------------------------------------------------

_IDENTIFIER = re.compile(r"[A-Za-z_]\w*\Z", re.ASCII)
_OPEN = "${"


def _spell(value: object) -> str:
    if isinstance(value, bool):
        return "true" if value else "false"
    return str(value)


def substitute(template: str, bindings: dict) -> str:
    """Fill every ``${name}`` from *bindings*; all other bytes pass through."""
    pieces = template.split(_OPEN)
    out = [pieces[0]]
    offset = len(pieces[0])
    for piece in pieces[1:]:
        close = piece.find("}")
        if close < 0:
            raise MalformedPlaceholder(f"unterminated placeholder at offset {offset}")
        name = piece[:close]
        if not _IDENTIFIER.match(name):
            raise MalformedPlaceholder(
                f"placeholder body {name!r} at offset {offset} is not an identifier")
        try:
            value = bindings[name]
        except KeyError:
            raise UnboundPlaceholder(name) from None
        out.append(_spell(value))
        out.append(piece[close + 1:])
        offset += len(_OPEN) + len(piece)
    return "".join(out)


# --- block templates -----------------------------------------------------------------

_TAG = re.compile(r"\{%\s*(.*?)\s*%\}", re.DOTALL)
_FOR = re.compile(r"for\s+([A-Za-z_]\w*)\s+in\s+(-?\w+)\s*\.\.\s*(-?\w+)\Z")
_IF = re.compile(r"if\s+(\S+)\Z")


class _Text:
    def __init__(self, text: str) -> None:
        self.text = text

    def expand(self, env: dict, out: list) -> None:
        try:
            out.append(substitute(self.text, env))
        except UnboundPlaceholder as exc:
            raise UnboundVariable(exc.name) from None


def _lookup(token: str, env: dict):
    if token not in env:
        raise UnboundVariable(token)
    return env[token]


class _Loop:
    def __init__(self, var: str, lo: str, hi: str, body: list) -> None:
        self.var, self.lo, self.hi, self.body = var, lo, hi, body

    @staticmethod
    def _bound(token: str, env: dict) -> int:
        if re.fullmatch(r"-?\d+", token):
            return int(token)
        value = _lookup(token, env)
        if isinstance(value, bool) or not isinstance(value, int):
            raise NonIntegerBound(f"loop bound {token!r} is {value!r}, not an integer")
        return value

    def expand(self, env: dict, out: list) -> None:
        for v in range(self._bound(self.lo, env), self._bound(self.hi, env)):
            inner = dict(env)
            inner[self.var] = v
            for node in self.body:
                node.expand(inner, out)


class _Cond:
    def __init__(self, cond: str, body: list) -> None:
        self.cond, self.body = cond, body

    def expand(self, env: dict, out: list) -> None:
        if self.cond in ("true", "false"):
            taken = self.cond == "true"
        else:
            taken = bool(_lookup(self.cond, env))
        if taken:
            for node in self.body:
                node.expand(env, out)


def _parse(template: str) -> list:
    """Build the block tree with an explicit stack (one frame per open tag)."""
    root: list = []
    stack: list[tuple[str, list]] = [("", root)]
    pos = 0
    for m in _TAG.finditer(template):
        if m.start() > pos:
            stack[-1][1].append(_Text(template[pos:m.start()]))
        pos = m.end()
        tag = m.group(1)
        if tag in ("endfor", "endif"):
            opener = stack[-1][0]
            if opener != tag[3:]:
                raise UnclosedBlock(f"unexpected {{% {tag} %}}")
            stack.pop()
            continue
        loop = _FOR.match(tag)
        if loop:
            node = _Loop(loop.group(1), loop.group(2), loop.group(3), [])
            stack[-1][1].append(node)
            stack.append(("for", node.body))
            continue
        cond = _IF.match(tag)
        if cond:
            node = _Cond(cond.group(1), [])
            stack[-1][1].append(node)
            stack.append(("if", node.body))
            continue
        raise UnclosedBlock(f"malformed block tag {{% {tag} %}}")
    if pos < len(template):
        stack[-1][1].append(_Text(template[pos:]))
    if len(stack) > 1:
        raise UnclosedBlock(f"missing {{% end{stack[-1][0]} %}}")
    return root


def render(template: str, context: dict | None = None) -> str:
    """Expand ``{% for %}`` / ``{% if %}`` blocks and ``${}`` placeholders."""
    out: list[str] = []
    env = dict(context or {})
    for node in _parse(template):
        node.expand(env, out)
    return "".join(out)


# --- syntax tree ------------------------------------------------------------------------


@dataclass(frozen=True)
class CType:
    """Scalar C type behind ``pointer`` levels of indirection."""

    base: str
    pointer: int = 0
    const: bool = False

    def render(self) -> str:
        head = ("const " if self.const else "") + self.base
        return head + (" " + "*" * self.pointer if self.pointer else "")

    def render_declarator(self, name: str) -> str:
        text = self.render()
        return text + name if self.pointer else f"{text} {name}"


class CNode:
    """Base of tree nodes.  Expression nodes implement ``_expr``; statement
    nodes implement ``_stmt``; a node may implement both."""

    __slots__ = ()

    def _expr(self, path: str) -> str:
        raise IllFormedTree(path, f"{type(self).__name__} is not an expression")

    def _stmt(self, lines: list, depth: int, path: str) -> None:
        raise IllFormedTree(path, f"{type(self).__name__} is not a statement")


_PAD = "    "


def _as_block(node, lines, depth, path):
    if not isinstance(node, Block):
        raise IllFormedTree(path, f"expected block, got {type(node).__name__}")
    node._stmt(lines, depth, path)


@dataclass(frozen=True)
class Raw(CNode):
    """Verbatim text in expression or statement position."""

    text: str

    def _expr(self, path):
        return self.text

    def _stmt(self, lines, depth, path):
        lines.extend((_PAD * depth + ln) if ln else ln for ln in self.text.splitlines())


@dataclass(frozen=True)
class Lit(CNode):
    text: str

    def __post_init__(self):
        if isinstance(self.text, int):
            object.__setattr__(self, "text", str(self.text))

    def _expr(self, path):
        return self.text


@dataclass(frozen=True)
class Ident(CNode):
    name: str

    def _expr(self, path):
        return self.name


@dataclass(frozen=True)
class Index(CNode):
    base: CNode
    index: CNode

    def _expr(self, path):
        return f"{_expr(self.base, path + '/index-base')}[{_expr(self.index, path + '/index')}]"


@dataclass(frozen=True)
class BinOp(CNode):
    op: str
    left: CNode
    right: CNode

    def _expr(self, path):
        def side(node, tag):
            text = _expr(node, f"{path}/{tag}")
            return f"({text})" if isinstance(node, BinOp) else text
        return f"{side(self.left, 'left')} {self.op} {side(self.right, 'right')}"


@dataclass(frozen=True)
class Call(CNode):
    func: str
    args: tuple = ()

    def _expr(self, path):
        inner = ", ".join(_expr(a, f"{path}/arg[{k}]") for k, a in enumerate(self.args))
        return f"{self.func}({inner})"

    def _stmt(self, lines, depth, path):
        lines.append(_PAD * depth + self._expr(path) + ";")


@dataclass(frozen=True)
class Assign(CNode):
    target: CNode
    value: CNode
    op: str = "="

    def _stmt(self, lines, depth, path):
        lhs = _expr(self.target, path + "/target")
        rhs = _expr(self.value, path + "/value")
        lines.append(f"{_PAD * depth}{lhs} {self.op} {rhs};")


@dataclass(frozen=True)
class Decl(CNode):
    ctype: CType
    name: str
    init: CNode | None = None

    def text(self, path: str) -> str:
        out = self.ctype.render_declarator(self.name)
        if self.init is not None:
            out += " = " + _expr(self.init, path + "/init")
        return out

    def _stmt(self, lines, depth, path):
        lines.append(_PAD * depth + self.text(path) + ";")


@dataclass(frozen=True)
class Block(CNode):
    stmts: tuple = ()

    def _stmt(self, lines, depth, path):
        for k, s in enumerate(self.stmts):
            _stmt(s, lines, depth, f"{path}/stmt[{k}]")


@dataclass(frozen=True)
class For(CNode):
    init: CNode | None
    cond: CNode | None
    step: CNode | None
    body: Block

    def _stmt(self, lines, depth, path):
        if self.init is None:
            init = ""
        elif isinstance(self.init, Decl):
            init = self.init.text(path + "/init")
        else:
            init = _expr(self.init, path + "/init")
        cond = "" if self.cond is None else _expr(self.cond, path + "/cond")
        step = "" if self.step is None else _expr(self.step, path + "/step")
        lines.append(f"{_PAD * depth}for ({init}; {cond}; {step}) {{")
        _as_block(self.body, lines, depth + 1, path + "/body")
        lines.append(_PAD * depth + "}")


@dataclass(frozen=True)
class If(CNode):
    cond: CNode
    then: Block
    orelse: Block | None = None

    def _stmt(self, lines, depth, path):
        lines.append(f"{_PAD * depth}if ({_expr(self.cond, path + '/cond')}) {{")
        _as_block(self.then, lines, depth + 1, path + "/then")
        if self.orelse is not None:
            lines.append(_PAD * depth + "} else {")
            _as_block(self.orelse, lines, depth + 1, path + "/else")
        lines.append(_PAD * depth + "}")


@dataclass(frozen=True)
class Param(CNode):
    ctype: CType
    name: str


@dataclass(frozen=True)
class FunctionDef(CNode):
    """A function; ``qualifiers`` prefixes the return type (e.g.
    ``extern "C" __global__``)."""

    name: str
    return_type: CType
    params: tuple
    body: Block
    qualifiers: str = ""

    def emit_into(self, lines: list, path: str) -> None:
        decls = []
        for k, p in enumerate(self.params):
            if not isinstance(p, Param):
                raise IllFormedTree(f"{path}/param[{k}]", "expected parameter")
            decls.append(p.ctype.render_declarator(p.name))
        head = (self.qualifiers + " " if self.qualifiers else "") + self.return_type.render()
        lines.append(f"{head} {self.name}({', '.join(decls)})")
        lines.append("{")
        _as_block(self.body, lines, 1, path + "/block")
        lines.append("}")


@dataclass(frozen=True)
class TranslationUnit(CNode):
    items: tuple = ()

    def emit_into(self, lines: list) -> None:
        path = "translation-unit"
        for k, item in enumerate(self.items):
            if isinstance(item, FunctionDef):
                if k:
                    lines.append("")
                item.emit_into(lines, f"{path}/function-def[{item.name}]")
            elif isinstance(item, (Raw, Decl)):
                item._stmt(lines, 0, f"{path}/item")
            else:
                raise IllFormedTree(path, f"{type(item).__name__} is not allowed at file scope")


def _expr(node, path: str) -> str:
    if not isinstance(node, CNode):
        raise IllFormedTree(path, f"{type(node).__name__} is not a CNode")
    return node._expr(path)


def _stmt(node, lines, depth, path) -> None:
    if not isinstance(node, CNode):
        raise IllFormedTree(path, f"{type(node).__name__} is not a CNode")
    node._stmt(lines, depth, path)


def counted_for(var: str, start: CNode, stop: CNode, body: Block,
                ctype: str = "int") -> For:
    """``for (<ctype> var = start; var < stop; ++var) body``."""
    return For(Decl(CType(ctype), var, start), BinOp("<", Ident(var), stop),
               Raw(f"++{var}"), body)


def emit(root: CNode) -> str:
    """Print *root* as source text; deterministic byte for byte.

    Expression roots return the bare expression; everything else returns
    newline-terminated lines.
    """
    lines: list[str] = []
    if isinstance(root, TranslationUnit):
        root.emit_into(lines)
    elif isinstance(root, FunctionDef):
        root.emit_into(lines, f"function-def[{root.name}]")
    elif isinstance(root, (Assign, Decl, For, If, Block, Raw, Call)):
        root._stmt(lines, 0, type(root).__name__.lower())
    elif isinstance(root, CNode):
        return root._expr(type(root).__name__.lower())
    else:
        raise IllFormedTree("root", f"{type(root).__name__} is not a CNode")
    return "\n".join(lines) + "\n"


# --- paper Fig. 4: unrolled vector addition, generated two ways -------------------
#
# The reference renders this as host C (src/csyntax.py:535-618); here both
# strategies emit the same sm_100a kernel: each thread handles `unroll`
# consecutive elements of a grid-stride walk, with a guarded remainder.

UNROLLED_ADD_CUDA = """\
extern "C" __global__ void ${name}(const ${ctype} *x, const ${ctype} *y, ${ctype} *z, long n)
{
    long i = ((long) blockIdx.x * blockDim.x + threadIdx.x) * ${unroll};
    const long step = (long) gridDim.x * blockDim.x * ${unroll};
    for (; i + ${unroll} <= n; i += step) {
{% for j in 0..unroll %}        z[i + ${j}] = x[i + ${j}] + y[i + ${j}];
{% endfor %}    }
{% if unrolled %}    for (long k = i; k < n && k < i + ${unroll}; ++k) {
        z[k] = x[k] + y[k];
    }
{% endif %}}
"""


# the reference's name for the Fig. 4a template (src/csyntax.py:535)
UNROLLED_ADD_TEMPLATE = UNROLLED_ADD_CUDA


def unrolled_add_template(unroll: int, ctype: str = "float", name: str = "vadd_unrolled") -> str:
    """Fig. 4a: the kernel rendered from the text template."""
    if unroll < 1:
        raise ValueError("unroll must be at least 1")
    return render(UNROLLED_ADD_CUDA, {"name": name, "ctype": ctype, "unroll": unroll,
                                      "unrolled": unroll > 1})


def unrolled_add_ast(unroll: int, ctype: str = "float",
                     name: str = "vadd_unrolled") -> TranslationUnit:
    """Fig. 4b: the same kernel built as a syntax tree (print with :func:`emit`)."""
    if unroll < 1:
        raise ValueError("unroll must be at least 1")

    def at(var: str, j: int) -> CNode:
        return Ident(var) if j == 0 else BinOp("+", Ident(var), Lit(j))

    def add(var: str, j: int) -> Assign:
        return Assign(Index(Ident("z"), at(var, j)),
                      BinOp("+", Index(Ident("x"), at(var, j)), Index(Ident("y"), at(var, j))))

    body: list = [
        Decl(CType("long"), "i", Raw(f"((long) blockIdx.x * blockDim.x + threadIdx.x) * {unroll}")),
        Decl(CType("long", const=True), "step", Raw(f"(long) gridDim.x * blockDim.x * {unroll}")),
        For(None, BinOp("<=", BinOp("+", Ident("i"), Lit(unroll)), Ident("n")),
            Raw("i += step"), Block(tuple(add("i", j) for j in range(unroll)))),
    ]
    if unroll > 1:
        body.append(For(Decl(CType("long"), "k", Ident("i")),
                        Raw(f"k < n && k < i + {unroll}"), Raw("++k"), Block((add("k", 0),))))
    fn = FunctionDef(name, CType("void"),
                     (Param(CType(ctype, pointer=1, const=True), "x"),
                      Param(CType(ctype, pointer=1, const=True), "y"),
                      Param(CType(ctype, pointer=1), "z"), Param(CType("long"), "n")),
                     Block(tuple(body)), qualifiers='extern "C" __global__')
    return TranslationUnit((fn,))
