"""Caffe-prototxt subset reader/writer (reference: prototxt.py:1-402).

Accepts the same grammar as the reference: protobuf text format with scalar
fields, repeated fields and nested messages (optional colon before ``{``),
``#`` comments, double-quoted strings with backslash escapes, numbers and
bare enum identifiers.  Unknown fields inside known messages are skipped
with a warning; unknown layer types raise ``UnknownLayerError``.  The layer
parameters produced are identical to the reference's (prototxt.py:232-326)
so compiled plans match.
"""

from __future__ import annotations

import logging
import re

from .errors import ParseError
from .netspec import DEFAULT_ELU_ALPHA, LayerKind, LayerSpec, NetworkSpec, layer_kind

log = logging.getLogger(__name__)

_TOKEN = re.compile(r'''
    (?P<nl>\n) |
    (?P<ws>[ \t\r]+) |
    (?P<comment>\#[^\n]*) |
    (?P<punct>[{}:,;]) |
    (?P<string>") |
    (?P<word>[^ \t\r\n\#"{}:,;]+)
''', re.VERBOSE)


def _lex(text: str):
    """Yield (kind, text, line, col) tokens, then ('eof', '', line, col)."""
    pos, line, line_start = 0, 1, 0
    n = len(text)
    while pos < n:
        m = _TOKEN.match(text, pos)
        kind = m.lastgroup
        col = pos - line_start + 1
        if kind == "nl":
            line += 1
            line_start = m.end()
        elif kind in ("ws", "comment"):
            pass
        elif kind == "string":
            j, buf = pos + 1, []
            while True:
                if j >= n or text[j] == "\n":
                    raise ParseError("unterminated string", line, col)
                ch = text[j]
                if ch == '"':
                    break
                if ch == "\\" and j + 1 < n:
                    buf.append(text[j + 1])
                    j += 2
                    continue
                buf.append(ch)
                j += 1
            yield ("string", "".join(buf), line, col)
            pos = j + 1
            continue
        elif kind == "punct":
            yield ("punct", m.group(), line, col)
        else:
            word = m.group()
            yield ("number" if word[0] in "+-.0123456789" else "ident", word, line, col)
        pos = m.end()
    yield ("eof", "", line, pos - line_start + 1)


class _Field:
    __slots__ = ("name", "value", "line")

    def __init__(self, name, value, line):
        self.name, self.value, self.line = name, value, line


def _number(text, line, col):
    body = text.lstrip("+-")
    try:
        if body.isdigit() or not any(c in text for c in ".eE"):
            return int(text)
        return float(text)
    except ValueError:
        raise ParseError("bad number %r" % text, line, col) from None


class _Reader:
    def __init__(self, text):
        self.toks = list(_lex(text))
        self.i = 0

    def peek(self):
        return self.toks[self.i]

    def take(self):
        t = self.toks[self.i]
        self.i += 1
        return t

    def message_body(self):
        out = []
        while True:
            kind, text, line, col = self.peek()
            if kind == "eof" or text == "}":
                return out
            if kind == "punct" and text in ",;":
                self.take()
                continue
            if kind != "ident":
                raise ParseError("expected a field name, got %r" % text, line, col)
            out.append(self.field())

    def field(self):
        _, name, line, _ = self.take()
        if self.peek()[1] == ":" and self.peek()[0] == "punct":
            self.take()
        kind, text, vline, vcol = self.peek()
        if kind == "punct" and text == "{":
            self.take()
            body = self.message_body()
            ck, ct, cl, cc = self.take()
            if ct != "}":
                raise ParseError("expected '}'", cl, cc)
            return _Field(name, body, line)
        self.take()
        if kind == "string" or kind == "ident":
            return _Field(name, text, line)
        if kind == "number":
            return _Field(name, _number(text, vline, vcol), line)
        raise ParseError("expected a value for field %r" % name, vline, vcol)

    def document(self):
        body = self.message_body()
        kind, text, line, col = self.peek()
        if kind != "eof":
            raise ParseError("unexpected %r" % text, line, col)
        return body


class _Msg:
    """Grouped view of a message body with typed accessors."""

    def __init__(self, fields, ctx):
        self.ctx = ctx
        self.groups: dict = {}
        for f in fields:
            self.groups.setdefault(f.name, []).append(f)

    def pop(self, key):
        return self.groups.pop(key, None)

    def scalar(self, f, typ):
        v = f.value
        if isinstance(v, list):
            raise ParseError("%s.%s is not a scalar" % (self.ctx, f.name), f.line)
        if typ is float and isinstance(v, int) and not isinstance(v, bool):
            v = float(v)
        if not isinstance(v, typ):
            raise ParseError("%s.%s expects %s, got %r" % (self.ctx, f.name, typ.__name__, f.value),
                             f.line)
        return v

    def one(self, key, typ, default=None, required_line=None):
        fs = self.pop(key)
        if not fs:
            if required_line is not None:
                raise ParseError("%s lacks %s" % (self.ctx, key), required_line)
            return default
        return self.scalar(fs[0], typ)

    def many(self, key, typ):
        return tuple(self.scalar(f, typ) for f in (self.pop(key) or []))

    def triple(self, key, default=None):
        fs = self.pop(key)
        if not fs:
            return default
        vals = [self.scalar(f, int) for f in fs]
        if len(vals) == 1:
            vals *= 3
        if len(vals) != 3:
            raise ParseError("%s.%s expects 1 or 3 values, got %d" % (self.ctx, key, len(fs)),
                             fs[0].line)
        return tuple(vals)

    def sub(self, key, line, required=True):
        fs = self.pop(key)
        if not fs:
            if required:
                raise ParseError("%s has no %s" % (self.ctx, key), line)
            return None
        f = fs[0]
        if not isinstance(f.value, list):
            raise ParseError("%s.%s must be a message" % (self.ctx, key), f.line)
        return _Msg(f.value, "%s.%s" % (self.ctx, key)), f.line

    def finish(self):
        for key, fs in self.groups.items():
            log.warning("line %d: skipping unknown field %s.%s", fs[0].line, self.ctx, key)


_ELTWISE = {"SUM": "add", "PROD": "mul", "DIV": "div"}
_POOL = {"MAX": "max", "AVE": "avg"}


def _layer(f: _Field) -> LayerSpec:
    if not isinstance(f.value, list):
        raise ParseError("layer must be a message", f.line)
    msg = _Msg(f.value, "layer")
    nf = msg.pop("name")
    if not nf:
        raise ParseError("layer without a name", f.line)
    name = msg.scalar(nf[0], str)
    msg.ctx = "layer %r" % name
    tf = msg.pop("type")
    if not tf:
        raise ParseError("%s has no type" % msg.ctx, f.line)
    kind = layer_kind(msg.scalar(tf[0], str))
    bottoms = msg.many("bottom", str)
    tops = msg.many("top", str)
    params: dict = {}
    if kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
        sub, sl = msg.sub("convolution_param", f.line)
        params["num_output"] = sub.one("num_output", int, required_line=sl)
        k = sub.triple("kernel_size")
        if k is None:
            raise ParseError("%s lacks kernel_size" % sub.ctx, sl)
        params["kernel"] = k
        params["stride"] = sub.triple("stride", (1, 1, 1))
        params["pad"] = sub.triple("pad", (0, 0, 0))
        sub.finish()
    elif kind is LayerKind.POOLING:
        sub, sl = msg.sub("pooling_param", f.line)
        mode = sub.one("pool", str, "MAX")
        if mode not in _POOL:
            raise ParseError("%s has unknown pool mode %r" % (sub.ctx, mode), sl)
        params["mode"] = _POOL[mode]
        w = sub.triple("kernel_size")
        if w is None:
            raise ParseError("%s lacks kernel_size" % sub.ctx, sl)
        params["window"] = w
        params["stride"] = sub.triple("stride", w)
        sub.finish()
    elif kind is LayerKind.ELTWISE:
        got = msg.sub("eltwise_param", f.line, required=False)
        op = "SUM"
        if got:
            sub, _ = got
            op = sub.one("operation", str, "SUM")
            sub.finish()
        if op not in _ELTWISE:
            raise ParseError("%s has unknown eltwise operation %r" % (msg.ctx, op), f.line)
        params["op"] = _ELTWISE[op]
    elif kind is LayerKind.ELU:
        got = msg.sub("elu_param", f.line, required=False)
        alpha = DEFAULT_ELU_ALPHA
        if got:
            sub, _ = got
            alpha = sub.one("alpha", float, DEFAULT_ELU_ALPHA)
            sub.finish()
        params["alpha"] = alpha
    elif kind is LayerKind.INPUT:
        sub, sl = msg.sub("input_param", f.line)
        shp, shl = sub.sub("shape", sl)
        dims = shp.many("dim", int)
        if len(dims) != 5:
            raise ParseError("%s expects 5 dims, got %d" % (shp.ctx, len(dims)), shl)
        params["shape"] = tuple(dims)
        sub.finish()
    msg.finish()
    return LayerSpec(name=name, kind=kind, bottoms=bottoms, tops=tops, params=params)


def parse_network(text: str) -> NetworkSpec:
    """Parse a network description and validate its wiring (prototxt.py:329-341)."""
    top = _Msg(_Reader(text).document(), "network")
    nf = top.pop("name")
    name = top.scalar(nf[0], str) if nf else "net"
    layers = tuple(_layer(f) for f in (top.pop("layer") or []))
    top.finish()
    spec = NetworkSpec(name=name, layers=layers)
    spec.validate()
    return spec


def _q(s: str) -> str:
    return '"' + s.replace("\\", "\\\\").replace('"', '\\"') + '"'


def print_network(spec: NetworkSpec) -> str:
    """Canonical text that parses back to an equal NetworkSpec."""
    out = ["name: " + _q(spec.name)]
    back_elt = {v: k for k, v in _ELTWISE.items()}
    back_pool = {v: k for k, v in _POOL.items()}
    for lay in spec.layers:
        p = lay.params
        body = ["name: " + _q(lay.name), "type: " + _q(lay.kind.value)]
        body += ["bottom: " + _q(b) for b in lay.bottoms]
        body += ["top: " + _q(t) for t in lay.tops]
        if lay.kind in (LayerKind.CONVOLUTION, LayerKind.DECONVOLUTION):
            inner = ["num_output: %d" % p["num_output"]]
            for key, src in (("kernel_size", "kernel"), ("stride", "stride"), ("pad", "pad")):
                inner += ["%s: %d" % (key, v) for v in p[src]]
            body += ["convolution_param {"] + ["  " + s for s in inner] + ["}"]
        elif lay.kind is LayerKind.POOLING:
            inner = ["pool: " + back_pool[p["mode"]]]
            inner += ["kernel_size: %d" % v for v in p["window"]]
            inner += ["stride: %d" % v for v in p["stride"]]
            body += ["pooling_param {"] + ["  " + s for s in inner] + ["}"]
        elif lay.kind is LayerKind.ELTWISE:
            body += ["eltwise_param {", "  operation: " + back_elt[p["op"]], "}"]
        elif lay.kind is LayerKind.ELU:
            body += ["elu_param {", "  alpha: %r" % float(p.get("alpha", DEFAULT_ELU_ALPHA)), "}"]
        elif lay.kind is LayerKind.INPUT:
            body += ["input_param {", "  shape {"] + ["    dim: %d" % d for d in p["shape"]]
            body += ["  }", "}"]
        out += ["layer {"] + ["  " + s for s in body] + ["}"]
    return "\n".join(out) + "\n"
