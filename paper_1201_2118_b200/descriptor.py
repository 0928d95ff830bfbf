"""Kernel descriptor front end: ``.ccl`` text -> raw kernels -> validated
descriptors -> execution plans and rendered headers.

Mirrors the reference's ``sforge::ccl`` (``inc/descriptor.hpp``) and the
plan/header part of ``sforge::codegen`` (``inc/codegen.hpp``): the same
grammar (descriptor.hpp:65-84), the same error texts and positions, the same
canonical rendering (descriptor.hpp:186-214), validation rules
(descriptor.hpp:287-373), plan (codegen.hpp:59-68), header
(codegen.hpp:86-126) and manifest (codegen.hpp:130-163). ``build_plan``
returns the ``ExecutionPlan`` that ``Simulation.register_kernel`` takes, so a
descriptor file drives the device kernels directly.

The parser is a small PEG interpreter over the descriptor grammar. Like the
reference's engine it records the farthest input position any terminal
examined and failed on, and a syntax error is reported there (line and
column counted as ``peg::line_col``, inc/peg.hpp:26-38), so error positions
agree with the reference's.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

from .sim import ExecutionPlan


class ParseError(Exception):
    """ccl::parse_error (descriptor.hpp:22-33): message plus line/column."""

    def __init__(self, what: str, line: int, column: int):
        super().__init__("%s at line %d, column %d" % (what, line, column))
        self.line, self.column = line, column


class DescriptorError(Exception):
    """ccl::descriptor_error (descriptor.hpp:35-38)."""


def line_col(text: str, offset: int) -> tuple[int, int]:
    offset = min(offset, len(text))
    line = 1 + text.count("\n", 0, offset)
    last = text.rfind("\n", 0, offset)
    return line, offset - last  # column is 1-based: offset - (last + 1) + 1


# ---- PEG interpreter ---------------------------------------------------------
# Expressions are tuples: ("lit", s) ("cls", [(lo, hi)...]) ("any",)
# ("seq", [e...]) ("alt", [e...]) ("star", e) ("opt", e) ("not", e) ("ref", name)

def _lit(s):
    return ("lit", s)


def _cls(*ranges):
    return ("cls", [(ord(a), ord(b)) for a, b in ranges])


def _seq(*e):
    return ("seq", list(e))


def _alt(*e):
    return ("alt", list(e))


def _star(e):
    return ("star", e)


def _opt(e):
    return ("opt", e)


def _not(e):
    return ("not", e)


def _ref(n):
    return ("ref", n)


_IDSTART = _cls(("A", "Z"), ("a", "z"), ("_", "_"))
_IDCHAR = _cls(("A", "Z"), ("a", "z"), ("0", "9"), ("_", "_"))
_WS, _IDENT, _STRING, _ATTRS, _NAMES = _ref("ws"), _ref("ident"), _ref("string"), _ref("attrs"), _ref("namelist")

# descriptor.hpp:65-84, rule for rule
_GRAMMAR = {
    "file": _seq(_WS, _star(_seq(_ref("kernel"), _WS))),
    "kernel": _seq(_lit("CCTK_CUDA_KERNEL"), _WS, _IDENT, _WS, _ATTRS, _lit("{"), _WS, _star(_ref("item")),
                   _lit("}")),
    "attrs": _star(_seq(_ref("attr"), _WS)),
    "attr": _seq(_ref("key"), _opt(_WS), _lit("="), _opt(_WS), _ref("value")),
    "key": _IDENT,
    "item": _alt(_ref("vargroup"), _ref("paramgroup")),
    "vargroup": _seq(_lit("CCTK_CUDA_KERNEL_VARIABLE"), _WS, _ATTRS, _lit("{"), _WS, _NAMES, _WS, _lit("}"), _WS,
                     _STRING, _WS),
    "paramgroup": _seq(_lit("CCTK_CUDA_KERNEL_PARAMETER"), _WS, _lit("{"), _WS, _NAMES, _WS, _lit("}"), _WS,
                       _STRING, _WS),
    "namelist": _seq(_IDENT, _star(_seq(_opt(_WS), _lit(","), _opt(_WS), _IDENT))),
    "value": _alt(_STRING, _ref("valtok")),
    "ident": _seq(_IDSTART, _star(_IDCHAR)),
    "valtok": _seq(_IDCHAR, _star(_IDCHAR)),
    "string": _seq(_lit('"'), _star(_seq(_not(_lit('"')), ("any",))), _lit('"')),
    "ws": _star(_alt(_ref("space"), _ref("comment"))),
    "space": _cls((" ", " "), ("\t", "\t"), ("\r", "\r"), ("\n", "\n")),
    "comment": _seq(_lit("#"), _star(_seq(_not(_cls(("\r", "\r"), ("\n", "\n"))), ("any",)))),
}


class _Node:
    __slots__ = ("rule", "begin", "end", "children")

    def __init__(self, rule, begin, end, children):
        self.rule, self.begin, self.end, self.children = rule, begin, end, children

    def named(self, rule):
        return [c for c in self.children if c.rule == rule]

    def first(self, rule):
        for c in self.children:
            if c.rule == rule:
                return c
        return None


class _Matcher:
    def __init__(self, text: str):
        self.t = text
        self.farthest = 0

    def fail(self, pos):
        if pos > self.farthest:
            self.farthest = pos

    def ev(self, e, pos, kids):
        """Returns the end position or None; appends rule nodes to kids."""
        k = e[0]
        t = self.t
        if k == "lit":
            s = e[1]
            for i, ch in enumerate(s):
                if pos + i >= len(t) or t[pos + i] != ch:
                    self.fail(pos + i)
                    return None
            return pos + len(s)
        if k == "cls":
            if pos < len(t):
                b = ord(t[pos])
                for lo, hi in e[1]:
                    if lo <= b <= hi:
                        return pos + 1
            self.fail(pos)
            return None
        if k == "any":
            if pos < len(t):
                return pos + 1
            self.fail(pos)
            return None
        if k == "seq":
            mark = len(kids)
            at = pos
            for c in e[1]:
                nxt = self.ev(c, at, kids)
                if nxt is None:
                    del kids[mark:]
                    return None
                at = nxt
            return at
        if k == "alt":
            for c in e[1]:
                mark = len(kids)
                nxt = self.ev(c, pos, kids)
                if nxt is not None:
                    return nxt
                del kids[mark:]
            return None
        if k == "star":
            at = pos
            while True:
                mark = len(kids)
                nxt = self.ev(e[1], at, kids)
                if nxt is None:
                    del kids[mark:]
                    return at
                if nxt == at:  # an empty iteration ends the repetition
                    return at
                at = nxt
        if k == "opt":
            mark = len(kids)
            nxt = self.ev(e[1], pos, kids)
            if nxt is None:
                del kids[mark:]
                return pos
            return nxt
        if k == "not":
            return None if self.ev(e[1], pos, []) is not None else pos
        if k == "ref":
            sub = []
            end = self.ev(_GRAMMAR[e[1]], pos, sub)
            if end is None:
                return None
            kids.append(_Node(e[1], pos, end, sub))
            return end
        raise AssertionError(k)

    def match(self, rule):
        kids = []
        end = self.ev(_ref(rule), 0, kids)
        return (kids[0] if kids else None), end


# ---- raw structure (descriptor.hpp:40-61) -------------------------------------

@dataclass
class AttrValue:
    text: str
    quoted: bool = False


@dataclass
class RawGroup:
    parameter: bool = False
    attrs: list = field(default_factory=list)  # [(key, AttrValue)]
    names: list = field(default_factory=list)
    description: str = ""


@dataclass
class RawKernel:
    name: str
    attrs: list = field(default_factory=list)
    groups: list = field(default_factory=list)


def _text(src, n):
    return src[n.begin:n.end]


def _read_attrs(src, attrs_node):
    out = []
    for a in attrs_node.named("attr"):
        key = a.first("key")
        ktext = _text(src, key)
        if any(k == ktext for k, _ in out):
            raise ParseError("duplicate attribute key '%s'" % ktext, *line_col(src, key.begin))
        v = a.first("value")
        s = v.first("string")
        out.append((ktext, AttrValue(_text(src, s)[1:-1], True) if s else AttrValue(_text(src, v.first("valtok")))))
    return out


def parse_descriptors(text: str) -> list[RawKernel]:
    """ccl::parse_descriptors (descriptor.hpp:148-182)."""
    m = _Matcher(text)
    root, end = m.match("file")
    if root is None or end != len(text):
        at = max(end, m.farthest) if root is not None else m.farthest
        raise ParseError("descriptor syntax error", *line_col(text, at))
    out = []
    for kn in root.named("kernel"):
        name = kn.first("ident")
        rk = RawKernel(_text(text, name))
        if any(p.name == rk.name for p in out):
            raise ParseError("kernel '%s' defined twice" % rk.name, *line_col(text, name.begin))
        rk.attrs = _read_attrs(text, kn.first("attrs"))
        for item in kn.named("item"):
            g = item.first("vargroup")
            rg = RawGroup()
            if g is None:
                g = item.first("paramgroup")
                rg.parameter = True
            else:
                rg.attrs = _read_attrs(text, g.first("attrs"))
            rg.names = [_text(text, i) for i in g.first("namelist").named("ident")]
            rg.description = _text(text, g.first("string"))[1:-1]
            rk.groups.append(rg)
        out.append(rk)
    return out


def render(kernels) -> str:
    """Canonical text (descriptor.hpp:186-214): parse(render(parse(t))) == parse(t)."""
    if isinstance(kernels, RawKernel):
        kernels = [kernels]

    def av(v):
        return '"%s"' % v.text if v.quoted else v.text

    parts = []
    for k in kernels:
        s = "CCTK_CUDA_KERNEL " + k.name + "\n"
        for key, v in k.attrs:
            s += "   " + key + "=" + av(v) + "\n"
        s += "{\n"
        for g in k.groups:
            s += "  CCTK_CUDA_KERNEL_PARAMETER" if g.parameter else "  CCTK_CUDA_KERNEL_VARIABLE"
            for key, v in g.attrs:
                s += " " + key + "=" + av(v)
            s += "\n  {\n    " + ", ".join(g.names) + "\n  } \"" + g.description + "\"\n"
        s += "}\n"
        parts.append(s)
    return "\n".join(parts)


# ---- validation (descriptor.hpp:217-373) --------------------------------------

INTENTS = ("IN", "OUT", "INOUT", "SEPARATEINOUT")


def readable(intent: str) -> bool:
    return intent != "OUT"


def writable(intent: str) -> bool:
    return intent != "IN"


@dataclass
class VariableBinding:
    name: str
    cached: bool = False
    intent: str = "IN"
    description: str = ""


@dataclass
class KernelDescriptor:
    name: str
    type: str = "3DBLOCK"
    stencil: tuple = (0, 0, 0, 0, 0, 0)  # -x +x -y +y -z +z
    tile: tuple = (0, 0, 0)
    variables: list = field(default_factory=list)
    parameters: list = field(default_factory=list)  # [(name, description)]


_LONG_MAX = 2 ** 63 - 1


def _from_chars(s: str):
    """std::from_chars for long over the whole token: optional '-', decimal digits."""
    body = s[1:] if s.startswith("-") else s
    if not body or not body.isascii() or not body.isdigit():
        return None
    v = int(s)
    return v if -_LONG_MAX - 1 <= v <= _LONG_MAX else None


def _int_list(kernel: str, attr: str, text: str):
    out = []
    at = 0
    while at <= len(text):
        comma = text.find(",", at)
        if comma < 0:
            comma = len(text)
        b, e = at, comma
        while b < e and text[b] in " \t":
            b += 1
        while e > b and text[e - 1] in " \t":
            e -= 1
        v = _from_chars(text[b:e])
        if v is None:
            raise DescriptorError("kernel '%s': %s entry is not an integer: '%s'" % (kernel, attr, text[at:comma]))
        out.append(v)
        if comma == len(text):
            break
        at = comma + 1
    return out


def _as_int(v: int) -> int:  # static_cast<int> of a long (two's complement wrap)
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= 1 << 31 else v


def validate(raw: RawKernel, known_fields: Iterable[str]) -> KernelDescriptor:
    """ccl::validate (descriptor.hpp:287-373)."""
    known = set(known_fields)
    k = KernelDescriptor(raw.name)
    saw = set()
    for key, v in raw.attrs:
        if key == "TYPE":
            saw.add(key)
            if v.text != "3DBLOCK":
                raise DescriptorError("kernel '%s': unsupported TYPE '%s'" % (k.name, v.text))
        elif key == "STENCIL":
            saw.add(key)
            vals = _int_list(k.name, "STENCIL", v.text)
            if len(vals) != 6:
                raise DescriptorError("kernel '%s': STENCIL needs 6 entries, got %d" % (k.name, len(vals)))
            if any(x < 0 for x in vals):
                raise DescriptorError("kernel '%s': STENCIL entries must be >= 0" % k.name)
            k.stencil = tuple(_as_int(x) for x in vals)
        elif key == "TILE":
            saw.add(key)
            vals = _int_list(k.name, "TILE", v.text)
            if len(vals) != 3:
                raise DescriptorError("kernel '%s': TILE needs 3 entries, got %d" % (k.name, len(vals)))
            if any(x < 1 for x in vals):
                raise DescriptorError("kernel '%s': TILE entries must be >= 1" % k.name)
            k.tile = tuple(_as_int(x) for x in vals)
        else:
            raise DescriptorError("kernel '%s': unknown attribute '%s'" % (k.name, key))
    for key in ("TYPE", "STENCIL", "TILE"):
        if key not in saw:
            raise DescriptorError("kernel '%s': missing %s" % (k.name, key))
    seen = set()
    for g in raw.groups:
        if g.parameter:
            for n in g.names:
                if n in seen:
                    raise DescriptorError("kernel '%s': name '%s' declared twice" % (k.name, n))
                seen.add(n)
                k.parameters.append((n, g.description))
            continue
        cached, intent = False, "IN"
        for key, v in g.attrs:
            if key == "CACHED":
                if v.text not in ("YES", "NO"):
                    raise DescriptorError("kernel '%s': CACHED must be YES or NO, got '%s'" % (k.name, v.text))
                cached = v.text == "YES"
            elif key == "INTENT":
                if v.text not in INTENTS:
                    raise DescriptorError("kernel '%s': bad INTENT '%s'" % (k.name, v.text))
                intent = v.text
            else:
                raise DescriptorError("kernel '%s': unknown variable attribute '%s'" % (k.name, key))
        for n in g.names:
            if n not in known:
                raise DescriptorError("kernel '%s': unknown variable '%s'" % (k.name, n))
            if n in seen:
                raise DescriptorError("kernel '%s': name '%s' declared twice" % (k.name, n))
            seen.add(n)
            k.variables.append(VariableBinding(n, cached, intent, g.description))
    return k


def validate_all(raw: Sequence[RawKernel], known_fields: Iterable[str]) -> list[KernelDescriptor]:
    known = set(known_fields)
    return [validate(r, known) for r in raw]


# ---- plans and headers (codegen.hpp) ----------------------------------------------

def build_plan(k: KernelDescriptor) -> ExecutionPlan:
    """codegen::build_plan (codegen.hpp:59-68): the plan Simulation.register_kernel takes."""
    return ExecutionPlan(kernel=k.name, tile=tuple(k.tile), halo=tuple(k.stencil),
                         bindings=tuple((v.name, v.intent, v.cached) for v in k.variables),
                         parameters=tuple(n for n, _ in k.parameters))


def render_header(k: KernelDescriptor, template: str = "3DBLOCK") -> tuple[str, list]:
    """codegen::render_header (codegen.hpp:86-126): (text, signature), the
    signature as [(name, "field" | "parameter" | "index")]."""
    if template != "3DBLOCK":
        raise ValueError("unsupported template for kernel '%s'" % k.name)
    n = k.name
    s = "/* Generated tile-kernel interface for %s.  Do not edit. */\n" % n
    s += "#ifndef SFORGE_GEN_%s_H\n#define SFORGE_GEN_%s_H\n\n" % (n, n)
    s += "/* template %s */\n" % template
    for a, ax in enumerate("XYZ"):
        s += "#define %s_TILE_%s %d\n" % (n, ax, k.tile[a])
    for a, ax in enumerate("XYZ"):
        s += "#define %s_HALO_%sL %d\n" % (n, ax, k.stencil[2 * a])
        s += "#define %s_HALO_%sH %d\n" % (n, ax, k.stencil[2 * a + 1])
    s += "\n"
    sig = []
    for v in k.variables:
        s += "/* %s: %s%s" % (v.name, v.intent, ", cached in tile-local storage */\n" if v.cached else " */\n")
        if readable(v.intent):
            s += "#define %s_LOAD_%s(di, dj, dk) SFORGE_FIELD_LOAD(%s, di, dj, dk)\n" % (n, v.name, v.name)
        if writable(v.intent):
            s += "#define %s_STORE_%s(value) SFORGE_FIELD_STORE(%s, value)\n" % (n, v.name, v.name)
        sig.append((v.name, "field"))
    for p, _ in k.parameters:
        s += "#define %s_PARAM_%s SFORGE_PARAM(%s)\n" % (n, p, p)
        sig.append((p, "parameter"))
    s += "#define %s_INDEX3 SFORGE_TILE_INDEX3()\n" % n
    sig.append(("INDEX3", "index"))
    s += "\n#endif\n"
    return s, sig


def manifest(kernels: Sequence[KernelDescriptor]) -> str:
    """The plans.txt manifest of codegen::write_generated (codegen.hpp:137-158)."""
    out = ""
    for k in kernels:
        p = build_plan(k)
        out += "kernel %s\n  template 3DBLOCK\n  tile %s\n  halo %s\n" % (
            k.name, " ".join(str(t) for t in p.tile), " ".join(str(h) for h in p.halo))
        for f, intent, cached in p.bindings:
            out += "  binding %s intent=%s cached=%s\n" % (f, intent, "YES" if cached else "NO")
        for prm in p.parameters:
            out += "  parameter %s\n" % prm
        out += "  header %s.h.generated\n\n" % k.name
    return out


def write_generated(kernels: Sequence[KernelDescriptor], directory: str) -> list[str]:
    """codegen::write_generated (codegen.hpp:130-163): one <kernel>.h.generated
    per descriptor plus plans.txt; returns the paths written."""
    os.makedirs(directory, exist_ok=True)
    written = []
    for k in kernels:
        path = os.path.join(directory, k.name + ".h.generated")
        with open(path, "w", newline="") as f:
            f.write(render_header(k)[0])
        written.append(path)
    path = os.path.join(directory, "plans.txt")
    with open(path, "w", newline="") as f:
        f.write(manifest(kernels))
    written.append(path)
    return written


def load_plans(text: str, known_fields: Iterable[str]) -> dict[str, ExecutionPlan]:
    """parse -> validate -> plan for every kernel of a descriptor file, by name."""
    return {k.name: build_plan(k) for k in validate_all(parse_descriptors(text), known_fields)}
