"""C-subset front end: AST node types, scanner and recursive-descent parser.

Behavioural contract (reference `pkg/src/acctuner/nodes.py:12-176` and
`pkg/src/acctuner/parser.py:86-535`):

* the accepted language is the reference subset -- `int|float|double`
  scalars and <=2-D arrays, assignments (`= += -= *= /=`), `++/--`, calls,
  `if/else`, `for`, `while`, `do ... while`, `return`, blocks;
* `//`, `/* */` comments and whole `#...` lines (inserted pragmas) are
  skipped, so an annotated program re-parses to the same loop tree;
* loops are numbered 0..n-1 in textual pre-order, the id being taken when
  the loop keyword is consumed;
* every node carries a 1-based line/col and 0-based byte offset, and every
  statement a byte span, because the emitter annotates the original text
  without reformatting it;
* anything outside the subset raises `ParseError` at the offending token
  with the reference's message text.

The implementation differs from the reference's: the scanner is a small
state machine over character classes and binary expressions use one
precedence-table loop instead of one method per level.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import ParseError

# --------------------------------------------------------------------------
# AST
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class SourcePos:
    line: int       # 1-based
    col: int        # 1-based
    offset: int     # 0-based byte offset


Span = tuple[int, int]  # [start, end) byte offsets


@dataclass(frozen=True)
class NumLit:
    value: float
    is_float: bool          # literal was written with '.', 'e' or 'E'
    pos: SourcePos


@dataclass(frozen=True)
class VarExpr:
    name: str
    pos: SourcePos


@dataclass(frozen=True)
class IndexExpr:
    name: str
    indices: tuple          # one or two index expressions
    pos: SourcePos


@dataclass(frozen=True)
class UnaryExpr:
    op: str                 # '!' or '-'
    operand: object
    pos: SourcePos


@dataclass(frozen=True)
class BinaryExpr:
    op: str
    left: object
    right: object
    pos: SourcePos          # position of the operator token


@dataclass(frozen=True)
class CallExpr:
    name: str
    args: tuple
    pos: SourcePos


@dataclass
class Decl:
    type_name: str
    name: str
    dims: tuple             # () for scalars; size expressions (None = unsized param)
    init: object | None
    pos: SourcePos
    span: Span

    @property
    def is_array(self) -> bool:
        return len(self.dims) > 0


@dataclass
class Assign:
    target: object          # VarExpr | IndexExpr
    op: str
    value: object
    pos: SourcePos
    span: Span


@dataclass
class IncDec:
    target: VarExpr
    op: str                 # '++' | '--'
    pos: SourcePos
    span: Span


@dataclass
class If:
    cond: object
    then_body: "Block"
    else_body: "Block | None"
    pos: SourcePos
    span: Span


@dataclass
class ForLoop:
    init: Assign | None
    cond: object | None
    step: Assign | IncDec | None
    body: "Block"
    loop_id: int
    pos: SourcePos
    span: Span


@dataclass
class WhileLoop:
    cond: object
    body: "Block"
    loop_id: int
    pos: SourcePos
    span: Span


@dataclass
class DoWhileLoop:
    body: "Block"
    cond: object
    loop_id: int
    pos: SourcePos
    span: Span


@dataclass
class CallStmt:
    call: CallExpr
    pos: SourcePos
    span: Span


@dataclass
class Return:
    value: object | None
    pos: SourcePos
    span: Span


@dataclass
class Block:
    statements: list
    pos: SourcePos
    span: Span


@dataclass
class Function:
    name: str
    return_type: str
    params: list
    body: Block
    pos: SourcePos
    span: Span


@dataclass
class Program:
    functions: list = field(default_factory=list)
    source_text: str = ""


LOOP_STMTS = (ForLoop, WhileLoop, DoWhileLoop)
LOOP_KIND = {ForLoop: "for", WhileLoop: "while", DoWhileLoop: "dowhile"}

# --------------------------------------------------------------------------
# Scanner
# --------------------------------------------------------------------------

TYPE_KEYWORDS = ("int", "float", "double")
KEYWORDS = TYPE_KEYWORDS + ("if", "else", "for", "while", "do", "return")
UNSUPPORTED_KEYWORDS = frozenset((
    "goto", "switch", "case", "default", "break", "continue", "struct",
    "union", "enum", "typedef", "void", "char", "long", "short", "unsigned",
    "signed", "static", "extern", "const", "sizeof"))
ASSIGN_OPS = ("=", "+=", "-=", "*=", "/=")

_TWO_CHAR = frozenset(("++", "--", "+=", "-=", "*=", "/=", "==", "!=", "<=",
                       ">=", "&&", "||"))
_ONE_CHAR = frozenset("+-*/%<>=!(){}[];,")


@dataclass(frozen=True)
class Token:
    kind: str           # 'ident' | 'num' | 'punct' | 'eof'
    text: str
    line: int
    col: int
    offset: int

    @property
    def pos(self) -> SourcePos:
        return SourcePos(self.line, self.col, self.offset)

    @property
    def end(self) -> int:
        return self.offset + len(self.text)


def _scan_number(text: str, start: int) -> int:
    """End offset of the numeric literal starting at `start`:
    digits [ '.' digit+ ] [ (e|E) [+-] digit+ ]."""
    n = len(text)
    j = start
    while j < n and text[j].isdigit():
        j += 1
    if j + 1 < n and text[j] == "." and text[j + 1].isdigit():
        j += 2
        while j < n and text[j].isdigit():
            j += 1
    if j < n and text[j] in "eE":
        k = j + 1
        if k < n and text[k] in "+-":
            k += 1
        if k < n and text[k].isdigit():
            while k < n and text[k].isdigit():
                k += 1
            j = k
    return j


def tokenize(text: str, path: str = "<source>") -> list[Token]:
    """Split source text into tokens, skipping blanks, comments and
    `#` lines.  Line/column bookkeeping follows the reference scanner
    exactly, including that skipping a `//` comment or a `#` line does not
    advance the column (the newline that ends it resets it)."""
    out: list[Token] = []
    n = len(text)
    pos = 0
    line = 1
    col = 1
    while pos < n:
        ch = text[pos]
        if ch == "\n":
            pos += 1
            line += 1
            col = 1
        elif ch in " \t\r":
            pos += 1
            col += 1
        elif ch == "#" or text.startswith("//", pos):
            nl = text.find("\n", pos)
            pos = n if nl < 0 else nl
        elif text.startswith("/*", pos):
            close = text.find("*/", pos + 2)
            if close < 0:
                raise ParseError("unterminated block comment", line, col, path)
            body = text[pos:close + 2]
            breaks = body.count("\n")
            if breaks:
                line += breaks
                col = len(body) - body.rfind("\n")
            else:
                col += len(body)
            pos = close + 2
        elif ch.isalpha() or ch == "_":
            end = pos + 1
            while end < n and (text[end].isalnum() or text[end] == "_"):
                end += 1
            out.append(Token("ident", text[pos:end], line, col, pos))
            col += end - pos
            pos = end
        elif ch.isdigit():
            end = _scan_number(text, pos)
            out.append(Token("num", text[pos:end], line, col, pos))
            col += end - pos
            pos = end
        elif text[pos:pos + 2] in _TWO_CHAR:
            out.append(Token("punct", text[pos:pos + 2], line, col, pos))
            pos += 2
            col += 2
        elif ch in _ONE_CHAR:
            out.append(Token("punct", ch, line, col, pos))
            pos += 1
            col += 1
        else:
            raise ParseError(f"unexpected character {ch!r}", line, col, path)
    out.append(Token("eof", "", line, col, n))
    return out


# --------------------------------------------------------------------------
# Parser
# --------------------------------------------------------------------------

# binary operator precedence, loosest first; every level is left-associative
_BINARY_LEVELS = (
    frozenset(("||",)),
    frozenset(("&&",)),
    frozenset(("==", "!=")),
    frozenset(("<", "<=", ">", ">=")),
    frozenset(("+", "-")),
    frozenset(("*", "/", "%")),
)


class _Cursor:
    """Token cursor plus the grammar.  One instance parses one text."""

    def __init__(self, text: str, path: str):
        self.text = text
        self.path = path
        self.toks = tokenize(text, path)
        self.k = 0
        self.loop_counter = 0

    # ---- cursor primitives ----
    def tok(self, ahead: int = 0) -> Token:
        return self.toks[min(self.k + ahead, len(self.toks) - 1)]

    def take(self) -> Token:
        t = self.toks[self.k]
        if t.kind != "eof":
            self.k += 1
        return t

    def looking_at(self, text: str) -> bool:
        t = self.tok()
        return t.text == text and t.kind in ("punct", "ident")

    def skip_if(self, text: str) -> Token | None:
        return self.take() if self.looking_at(text) else None

    def fail(self, message: str, at: Token | None = None):
        at = at if at is not None else self.tok()
        raise ParseError(message, at.line, at.col, self.path)

    def need(self, text: str) -> Token:
        t = self.tok()
        if t.text != text:
            shown = repr(t.text) if t.text else "end of input"
            self.fail(f"expected {text!r}, found {shown}", t)
        return self.take()

    def reject_unsupported(self, t: Token):
        if t.kind == "ident" and t.text in UNSUPPORTED_KEYWORDS:
            self.fail(f"unsupported construct {t.text!r}", t)

    def identifier(self) -> Token:
        t = self.tok()
        self.reject_unsupported(t)
        if t.kind != "ident" or t.text in KEYWORDS:
            self.fail(f"expected identifier, found {t.text!r}", t)
        return self.take()

    def last_end(self) -> int:
        return self.toks[self.k - 1].end

    def next_loop_id(self) -> int:
        lid = self.loop_counter
        self.loop_counter += 1
        return lid

    # ---- declarations ----
    def program(self) -> Program:
        fns = []
        while self.tok().kind != "eof":
            fns.append(self.function())
        return Program(fns, self.text)

    def function(self) -> Function:
        head = self.tok()
        self.reject_unsupported(head)
        if head.text not in TYPE_KEYWORDS:
            self.fail(f"expected a function definition, found {head.text!r}", head)
        self.take()
        name = self.identifier()
        self.need("(")
        params = []
        if not self.looking_at(")"):
            params.append(self.parameter())
            while self.skip_if(","):
                params.append(self.parameter())
        self.need(")")
        body = self.block()
        return Function(name.text, head.text, params, body, head.pos,
                        (head.offset, body.span[1]))

    def parameter(self) -> Decl:
        ty = self.tok()
        self.reject_unsupported(ty)
        if ty.text not in TYPE_KEYWORDS:
            self.fail(f"expected parameter type, found {ty.text!r}", ty)
        self.take()
        name = self.identifier()
        dims = self.dimensions(sized=False)
        return Decl(ty.text, name.text, dims, None, name.pos, (ty.offset, self.last_end()))

    def dimensions(self, sized: bool) -> tuple:
        dims: list = []
        while self.looking_at("["):
            self.take()
            if self.looking_at("]"):
                if sized:
                    self.fail("array dimension requires a size expression")
                dims.append(None)
            else:
                dims.append(self.expression())
            self.need("]")
            if len(dims) > 2:
                self.fail("arrays of more than two dimensions are not supported")
        return tuple(dims)

    def declaration(self):
        ty = self.take()
        decls = [self.declarator(ty)]
        while self.skip_if(","):
            decls.append(self.declarator(ty))
        semi = self.need(";")
        for d in decls:
            d.span = (d.span[0], semi.end)
        return decls if len(decls) > 1 else decls[0]

    def declarator(self, ty: Token) -> Decl:
        name = self.identifier()
        dims = self.dimensions(sized=True)
        init = None
        if self.skip_if("="):
            if dims:
                self.fail("array initializers are not supported", name)
            init = self.expression()
        return Decl(ty.text, name.text, dims, init, name.pos, (ty.offset, self.last_end()))

    # ---- statements ----
    def block(self) -> Block:
        lbrace = self.need("{")
        stmts: list = []
        while not self.looking_at("}"):
            if self.tok().kind == "eof":
                self.fail("unterminated block; expected '}'")
            s = self.statement()
            if isinstance(s, list):
                stmts.extend(s)
            else:
                stmts.append(s)
        rbrace = self.need("}")
        return Block(stmts, lbrace.pos, (lbrace.offset, rbrace.end))

    def statement(self):
        t = self.tok()
        self.reject_unsupported(t)
        word = t.text
        if word in TYPE_KEYWORDS:
            return self.declaration()
        handler = {
            "if": self.if_stmt, "for": self.for_stmt, "while": self.while_stmt,
            "do": self.do_stmt, "return": self.return_stmt, "{": self.block,
        }.get(word)
        if handler is not None:
            return handler()
        if t.kind == "ident":
            return self.simple_stmt()
        self.fail(f"expected a statement, found {word!r}", t)

    def simple_stmt(self):
        first = self.tok()
        if self.tok(1).text == "(":
            call = self.primary()
            if not isinstance(call, CallExpr):
                self.fail("expected a call statement", first)
            semi = self.need(";")
            return CallStmt(call, first.pos, (first.offset, semi.end))
        s = self.assignment()
        semi = self.need(";")
        s.span = (s.span[0], semi.end)
        return s

    def index_list(self, anchor: Token) -> tuple:
        idx = []
        while self.looking_at("["):
            self.take()
            idx.append(self.expression())
            self.need("]")
        if len(idx) > 2:
            self.fail("arrays of more than two dimensions are not supported", anchor)
        return tuple(idx)

    def assignment(self):
        first = self.tok()
        name = self.identifier()
        if self.tok().text in ("++", "--"):
            op = self.take()
            return IncDec(VarExpr(name.text, name.pos), op.text, first.pos,
                          (first.offset, op.end))
        if self.looking_at("["):
            target = IndexExpr(name.text, self.index_list(first), name.pos)
        else:
            target = VarExpr(name.text, name.pos)
        op = self.tok()
        if op.text not in ASSIGN_OPS:
            self.fail(f"expected an assignment operator, found {op.text!r}", op)
        self.take()
        value = self.expression()
        return Assign(target, op.text, value, first.pos, (first.offset, self.last_end()))

    def body(self) -> Block:
        if self.looking_at("{"):
            return self.block()
        s = self.statement()
        if isinstance(s, list):
            return Block(s, s[0].pos, (s[0].span[0], s[-1].span[1]))
        return Block([s], s.pos, s.span)

    def if_stmt(self) -> If:
        kw = self.need("if")
        self.need("(")
        cond = self.expression()
        self.need(")")
        then_body = self.body()
        else_body = self.body() if self.skip_if("else") else None
        last = else_body if else_body is not None else then_body
        return If(cond, then_body, else_body, kw.pos, (kw.offset, last.span[1]))

    def for_stmt(self) -> ForLoop:
        kw = self.need("for")
        lid = self.next_loop_id()
        self.need("(")
        init = None
        if not self.looking_at(";"):
            init = self.assignment()
            if isinstance(init, IncDec):
                self.fail("for-loop initializer must be an assignment", kw)
        self.need(";")
        cond = None if self.looking_at(";") else self.expression()
        self.need(";")
        step = None if self.looking_at(")") else self.assignment()
        self.need(")")
        body = self.body()
        return ForLoop(init, cond, step, body, lid, kw.pos, (kw.offset, body.span[1]))

    def while_stmt(self) -> WhileLoop:
        kw = self.need("while")
        lid = self.next_loop_id()
        self.need("(")
        cond = self.expression()
        self.need(")")
        body = self.body()
        return WhileLoop(cond, body, lid, kw.pos, (kw.offset, body.span[1]))

    def do_stmt(self) -> DoWhileLoop:
        kw = self.need("do")
        lid = self.next_loop_id()
        body = self.body()
        self.need("while")
        self.need("(")
        cond = self.expression()
        self.need(")")
        semi = self.need(";")
        return DoWhileLoop(body, cond, lid, kw.pos, (kw.offset, semi.end))

    def return_stmt(self) -> Return:
        kw = self.need("return")
        value = None if self.looking_at(";") else self.expression()
        semi = self.need(";")
        return Return(value, kw.pos, (kw.offset, semi.end))

    # ---- expressions ----
    def expression(self, level: int = 0):
        if level == len(_BINARY_LEVELS):
            return self.unary()
        ops = _BINARY_LEVELS[level]
        left = self.expression(level + 1)
        while self.tok().kind == "punct" and self.tok().text in ops:
            op = self.take()
            right = self.expression(level + 1)
            left = BinaryExpr(op.text, left, right, op.pos)
        return left

    def unary(self):
        t = self.tok()
        if t.kind == "punct" and t.text in ("!", "-"):
            self.take()
            return UnaryExpr(t.text, self.unary(), t.pos)
        return self.primary()

    def primary(self):
        t = self.tok()
        self.reject_unsupported(t)
        if t.kind == "num":
            self.take()
            floaty = any(c in t.text for c in ".eE")
            return NumLit(float(t.text), floaty, t.pos)
        if t.text == "(":
            self.take()
            inner = self.expression()
            self.need(")")
            return inner
        if t.kind == "ident" and t.text not in KEYWORDS:
            self.take()
            if self.looking_at("("):
                self.take()
                args = []
                if not self.looking_at(")"):
                    args.append(self.expression())
                    while self.skip_if(","):
                        args.append(self.expression())
                self.need(")")
                return CallExpr(t.text, tuple(args), t.pos)
            if self.looking_at("["):
                return IndexExpr(t.text, self.index_list(t), t.pos)
            return VarExpr(t.text, t.pos)
        self.fail(f"expected an expression, found {t.text!r}", t)


def parse(text: str, path: str = "<source>") -> Program:
    """Parse C-subset source into a Program (reference `parser.py:528-535`).

    Empty input gives a Program with no functions; anything outside the
    subset raises ParseError at the offending token."""
    return _Cursor(text, path).program()
