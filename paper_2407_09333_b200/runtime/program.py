"""Lowered hash programs: the subset of the reference's lowered IR the B200
runtime executes, as plain records.

The reference compiles ``crypto.hash_batch`` through ``lower-crypto`` and
``lower-hyper-for`` into a flat op list (``pkg/src/hetoc/passes/
lower_hyper_for.py:279-368``): per device binding one launch group of
``hyper.alloc`` (with ``slice_stride``), ``hyper.memcpy`` (element offsets),
``dev.launch`` over the local range with the global ``offset``, and the
copy-back / ``hyper.dealloc`` tail.  This module holds that op list
(:class:`Program`), renders it in the reference printer's canonical text
(``pkg/src/hetoc/hir/printer.py``), parses that text back, and converts a
reference ``HirModule`` object (duck-typed; ``pkg/src/hetoc/hir/core.py:108-150``)
so a lowered module can be handed to :mod:`.executor` either as an object or
as its printed form.

Only the ops the lowering emits for hash workloads are representable:
``const addi muli memref.alloc memref.dealloc memref.copy hyper.alloc
hyper.dealloc hyper.memcpy par.loop dev.launch return`` at top level, and the
canonical digest loop body (``crypto.digest`` on the induction variable, or on
``iv + const`` -- ``_match_digest_loop``, ``executor.py:240-259``).

Variable-length batches add one loop body the reference
compiler cannot emit -- its ``crypto.hash_batch`` requires ``msg_len``
(``pkg/src/hetoc/hir/verify.py:343-358``) and its lowering uses fixed strides
(``pkg/src/hetoc/passes/lower_crypto.py:35-78``):

    crypto.digest_varlen %msgs, %offsets, %out, %iv {alg="md5", offset_base=B}

message ``iv`` is ``msgs[offsets[iv] - B, offsets[iv+1] - B)``: the offsets
slice copied to a device keeps the batch's global byte offsets and ``B`` (the
first offset of the slice) re-bases them onto the device's data slice.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

ELEM_BYTES = {"i8": 1, "i32": 4, "i64": 8, "index": 8, "f64": 8}
TOP_LEVEL = ("const", "addi", "muli", "memref.alloc", "memref.dealloc", "memref.copy", "hyper.alloc",
             "hyper.dealloc", "hyper.memcpy", "par.loop", "dev.launch", "return")


class ProgramError(ValueError):
    pass


@dataclass(frozen=True)
class BufType:
    elem: str
    length: int
    space: str = "host"

    @property
    def nbytes(self) -> int:
        return self.length * ELEM_BYTES[self.elem]

    def __str__(self) -> str:  # printer.py Buffer.__str__ (core.py:38-41)
        if self.space == "host":
            return f"buf<{self.elem}, {self.length}>"
        return f'buf<{self.elem}, {self.length}, "{self.space}">'


@dataclass(frozen=True)
class DigestLoop:
    """The canonical digest loop body: rows [lb + base, ub + base) of ``msgs``
    hashed into ``out``; ``from_const`` says the base came from the
    global-offset preamble (so batched sub-ranges shift it)."""

    msgs: int
    out: int
    alg: str
    msg_len: int
    accel: bool
    base: int = 0
    from_const: bool = False


@dataclass(frozen=True)
class VarDigestLoop:
    """The variable-length digest loop body: message t of the launch range is
    ``msgs[offsets[t] - offset_base, offsets[t+1] - offset_base)`` (``offsets``
    an i64 buffer of n+1 global byte offsets), digest into ``out`` row t."""

    msgs: int
    offsets: int
    out: int
    alg: str
    offset_base: int
    base: int = 0
    from_const: bool = False


@dataclass
class Op:
    opcode: str
    operands: list[int] = field(default_factory=list)  # value ids
    result: int | None = None
    attrs: dict = field(default_factory=dict)
    body: DigestLoop | VarDigestLoop | None = None  # par.loop / dev.launch
    rtype: object = None  # BufType for allocs, scalar kind for const/addi/muli


@dataclass
class Program:
    name: str
    params: list[tuple[int, BufType]]
    ops: list[Op]
    param_names: list[str] | None = None

    def names(self) -> list[str]:
        return list(self.param_names) if self.param_names else [f"arg{i}" for i in range(len(self.params))]

    # ---------------------------------------------------------------- printer
    def format(self) -> str:
        """The reference printer's canonical text (printer.py:104-236), values
        renumbered densely in definition order."""
        ids: dict = {}

        def define(v) -> str:
            ids[v] = len(ids)
            return f"%{ids[v]}"

        def ref(v: int) -> str:
            return f"%{ids[v]}"

        lines = ["func @%s(%s) {" % (self.name, ", ".join(f"{define(v)}: {t}" for v, t in self.params))]
        for op in self.ops:
            lines.extend("  " + ln for ln in _format_op(op, define, ref))
        lines.append("}")
        return "\n".join(lines) + "\n"


def _attr_value(v) -> str:  # printer.py:18-23
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (int, float)):
        return repr(v)
    return f'"{v}"'


def _attr_dict(attrs: dict, skip=()) -> str:
    items = [(k, v) for k, v in sorted(attrs.items()) if k not in skip]
    return "" if not items else " {" + ", ".join(f"{k}={_attr_value(v)}" for k, v in items) + "}"


def _format_op(op: Op, define, ref) -> list[str]:
    o = op.opcode
    if o == "const":
        return [f"{define(op.result)} = const {_attr_value(op.attrs['value'])} : {op.rtype}"]
    if o in ("addi", "muli"):
        a, b = (ref(x) for x in op.operands)
        return [f"{define(op.result)} = {o} {a}, {b} : {op.rtype}"]
    if o == "memref.alloc":
        return [f"{define(op.result)} = memref.alloc : {op.rtype}"]
    if o == "hyper.alloc":
        t = BufType(op.rtype.elem, op.rtype.length)
        return [f'{define(op.result)} = hyper.alloc dev("{op.attrs["device"]}"){_attr_dict(op.attrs, ("device",))} : {t}']
    if o in ("hyper.dealloc", "memref.dealloc"):
        return [f"{o} {ref(op.operands[0])}{_attr_dict(op.attrs)}"]
    if o == "memref.copy":
        return [f"memref.copy {ref(op.operands[0])}, {ref(op.operands[1])}"]
    if o == "hyper.memcpy":
        return [f"hyper.memcpy {ref(op.operands[0])}, {ref(op.operands[1])}{_attr_dict(op.attrs)}"]
    if o in ("par.loop", "dev.launch"):
        iv = define(op.result)
        head = f"{o} {iv} = {op.attrs['lb']} to {op.attrs['ub']} device(\"{op.attrs['device']}\")"
        if o == "dev.launch":
            head += f" offset({op.attrs.get('offset', 0)})"
            if "group" in op.attrs:
                head += f" group({op.attrs['group']})"
        d = op.body
        inner = []
        idx = iv
        if d.from_const:
            c = define(("const", id(op)))  # the preamble's values have no ids of their own
            g = define(("addi", id(op)))
            inner += [f"{c} = const {d.base} : index", f"{g} = addi {iv}, {c} : index"]
            idx = g
        if isinstance(d, VarDigestLoop):
            attrs = {"alg": d.alg, "offset_base": d.offset_base}
            inner += [f"crypto.digest_varlen {ref(d.msgs)}, {ref(d.offsets)}, {ref(d.out)}, {idx}{_attr_dict(attrs)}",
                      "yield"]
        else:
            attrs = {"accel": d.accel, "alg": d.alg, "msg_len": d.msg_len}
            inner += [f"crypto.digest {ref(d.msgs)}, {ref(d.out)}, {idx}{_attr_dict(attrs)}", "yield"]
        return [head + " {"] + ["  " + x for x in inner] + ["}"]
    if o == "return":
        return ["return"]
    raise ProgramError(f"cannot print opcode '{o}'")


# -------------------------------------------------------------------- parser
_BUF = r'buf<(\w+), (\d+)(?:, "([^"]*)")?>'
_RE_FUNC = re.compile(r"^func @(\w+)\((.*)\) \{$")
_RE_PARAM = re.compile(r"%(\d+): " + _BUF)
_RE_CONST = re.compile(r"^%(\d+) = const (\S+) : (\w+)$")
_RE_BIN = re.compile(r"^%(\d+) = (addi|muli) %(\d+), %(\d+) : (\w+)$")
_RE_MALLOC = re.compile(r"^%(\d+) = memref\.alloc : " + _BUF + "$")
_RE_HALLOC = re.compile(r'^%(\d+) = hyper\.alloc dev\("([^"]+)"\)(?: \{(.*)\})? : ' + _BUF + "$")
_RE_DEALLOC = re.compile(r"^(hyper\.dealloc|memref\.dealloc) %(\d+)(?: \{(.*)\})?$")
_RE_MCOPY = re.compile(r"^memref\.copy %(\d+), %(\d+)$")
_RE_HCOPY = re.compile(r"^hyper\.memcpy %(\d+), %(\d+)(?: \{(.*)\})?$")
_RE_LOOP = re.compile(r'^(par\.loop|dev\.launch) %(\d+) = (-?\d+) to (-?\d+) device\("([^"]+)"\)'
                      r"(?: offset\((-?\d+)\))?(?: group\((\d+)\))? \{$")
_RE_DIGEST = re.compile(r"^crypto\.digest %(\d+), %(\d+), %(\d+)(?: \{(.*)\})?$")
_RE_VDIGEST = re.compile(r"^crypto\.digest_varlen %(\d+), %(\d+), %(\d+), %(\d+)(?: \{(.*)\})?$")


def _parse_scalar(tok: str):
    if tok in ("true", "false"):
        return tok == "true"
    if tok.startswith('"'):
        return tok[1:-1]
    try:
        return int(tok)
    except ValueError:
        return float(tok)


def _parse_attrs(s: str | None) -> dict:
    if not s:
        return {}
    out = {}
    for part in s.split(", "):
        k, _, v = part.partition("=")
        out[k.strip()] = _parse_scalar(v.strip())
    return out


def parse(text: str, param_names: list[str] | None = None) -> Program:
    """Parse the reference printer's text of a lowered hash program."""
    lines = [ln.strip() for ln in text.strip().splitlines() if ln.strip()]
    if not lines:
        raise ProgramError("empty program")
    m = _RE_FUNC.match(lines[0])
    if not m:
        raise ProgramError(f"line 1: expected 'func @name(...) {{', got {lines[0]!r}")
    name = m.group(1)
    params = []
    for pm in _RE_PARAM.finditer(m.group(2)):
        params.append((int(pm.group(1)), BufType(pm.group(2), int(pm.group(3)), pm.group(4) or "host")))
    ops: list[Op] = []
    i = 1
    while i < len(lines):
        ln = lines[i]
        where = f"line {i + 1}"
        if ln == "}":
            if i != len(lines) - 1:
                raise ProgramError(f"{where}: text after the end of the function")
            break
        if ln == "return":
            ops.append(Op("return"))
        elif m := _RE_CONST.match(ln):
            ops.append(Op("const", [], int(m.group(1)), {"value": _parse_scalar(m.group(2))}, rtype=m.group(3)))
        elif m := _RE_BIN.match(ln):
            ops.append(Op(m.group(2), [int(m.group(3)), int(m.group(4))], int(m.group(1)), rtype=m.group(5)))
        elif m := _RE_MALLOC.match(ln):
            ops.append(Op("memref.alloc", [], int(m.group(1)), {},
                          rtype=BufType(m.group(2), int(m.group(3)), m.group(4) or "host")))
        elif m := _RE_HALLOC.match(ln):
            attrs = _parse_attrs(m.group(3))
            attrs["device"] = m.group(2)
            ops.append(Op("hyper.alloc", [], int(m.group(1)), attrs,
                          rtype=BufType(m.group(4), int(m.group(5)), m.group(2))))
        elif m := _RE_DEALLOC.match(ln):
            ops.append(Op(m.group(1), [int(m.group(2))], None, _parse_attrs(m.group(3))))
        elif m := _RE_MCOPY.match(ln):
            ops.append(Op("memref.copy", [int(m.group(1)), int(m.group(2))]))
        elif m := _RE_HCOPY.match(ln):
            ops.append(Op("hyper.memcpy", [int(m.group(1)), int(m.group(2))], None, _parse_attrs(m.group(3))))
        elif m := _RE_LOOP.match(ln):
            opcode, iv = m.group(1), int(m.group(2))
            attrs = {"lb": int(m.group(3)), "ub": int(m.group(4)), "device": m.group(5)}
            if opcode == "dev.launch":
                attrs["offset"] = int(m.group(6) or 0)
                if m.group(7) is not None:
                    attrs["group"] = int(m.group(7))
            body = []
            i += 1
            while i < len(lines) and lines[i] != "}":
                body.append(lines[i])
                i += 1
            if i == len(lines):
                raise ProgramError(f"{where}: unterminated loop body")
            ops.append(Op(opcode, [], iv, attrs, body=_parse_digest_body(body, iv, where)))
        else:
            raise ProgramError(f"{where}: unsupported op {ln!r} (the B200 runtime executes lowered hash programs)")
        i += 1
    return Program(name, params, ops, param_names)


def _parse_digest_body(body: list[str], iv: int, where: str) -> DigestLoop | VarDigestLoop:
    """Recognise the canonical digest loop (executor.py:240-259) in text."""
    if len(body) == 2 and (m := _RE_VDIGEST.match(body[0])) and body[1] == "yield" and int(m.group(4)) == iv:
        a = _parse_attrs(m.group(5))
        return VarDigestLoop(int(m.group(1)), int(m.group(2)), int(m.group(3)), a["alg"], int(a["offset_base"]))
    if len(body) == 4 and body[3] == "yield" and (v := _RE_VDIGEST.match(body[2])):
        c, add = _RE_CONST.match(body[0]), _RE_BIN.match(body[1])
        if c and add and add.group(2) == "addi" and int(v.group(4)) == int(add.group(1)) and \
                {int(add.group(3)), int(add.group(4))} == {iv, int(c.group(1))}:
            a = _parse_attrs(v.group(5))
            return VarDigestLoop(int(v.group(1)), int(v.group(2)), int(v.group(3)), a["alg"], int(a["offset_base"]),
                                 int(_parse_scalar(c.group(2))), True)
    if len(body) == 2 and (m := _RE_DIGEST.match(body[0])) and body[1] == "yield" and int(m.group(3)) == iv:
        a = _parse_attrs(m.group(4))
        return DigestLoop(int(m.group(1)), int(m.group(2)), a["alg"], int(a["msg_len"]), bool(a.get("accel")))
    if len(body) == 4 and body[3] == "yield":
        c, add, dig = _RE_CONST.match(body[0]), _RE_BIN.match(body[1]), _RE_DIGEST.match(body[2])
        if c and add and dig and add.group(2) == "addi" and int(dig.group(3)) == int(add.group(1)):
            ops = {int(add.group(3)), int(add.group(4))}
            if ops == {iv, int(c.group(1))}:
                a = _parse_attrs(dig.group(4))
                return DigestLoop(int(dig.group(1)), int(dig.group(2)), a["alg"], int(a["msg_len"]),
                                  bool(a.get("accel")), int(_parse_scalar(c.group(2))), True)
    raise ProgramError(f"{where}: loop body is not the canonical crypto.digest loop")


# --------------------------------------------------- reference object adapter
def from_hir(module, function: str = "main") -> Program:
    """Convert a lowered reference ``HirModule`` (duck-typed: ``functions``,
    ``Function.params/body/param_names``, ``HirOp.opcode/operands/results/
    attrs/regions``) into a :class:`Program`."""
    funcs = [f for f in module.functions if f.name == function]
    if not funcs:
        raise ProgramError(f"no function @{function}")
    func = funcs[0]
    vid: dict[int, int] = {}

    def v(x) -> int:
        if id(x) not in vid:
            vid[id(x)] = len(vid)
        return vid[id(x)]

    def btype(t) -> BufType:
        return BufType(t.elem, int(t.length), getattr(t, "space", "host"))

    params = [(v(p), btype(p.type)) for p in func.params]
    ops: list[Op] = []
    for op in func.body.ops:
        o = op.opcode
        if o not in TOP_LEVEL:
            raise ProgramError(f"unsupported top-level op '{o}' (the B200 runtime executes lowered hash programs)")
        res = v(op.results[0]) if op.results and o not in ("par.loop", "dev.launch") else None
        attrs = dict(op.attrs)
        rtype = None
        if o in ("memref.alloc", "hyper.alloc"):
            rtype = btype(op.results[0].type)
        elif o in ("const", "addi", "muli"):
            rtype = op.results[0].type.kind
        body = None
        if o in ("par.loop", "dev.launch"):
            if op.results:
                raise ProgramError("loop results must be lowered away (run lower-reduce)")
            block = op.regions[0].blocks[0]
            res = v(block.args[0])
            body = _digest_from_block(block, v)
        ops.append(Op(o, [v(x) for x in op.operands], res, attrs, body=body, rtype=rtype))
    return Program(func.name, params, ops, list(func.param_names) if getattr(func, "param_names", None) else None)


def _digest_from_block(block, v) -> DigestLoop:
    ops, iv = block.ops, block.args[0]
    codes = [o.opcode for o in ops]
    if codes == ["crypto.digest", "yield"] and ops[0].operands[2] is iv:
        d = ops[0]
        return DigestLoop(v(d.operands[0]), v(d.operands[1]), d.attrs["alg"], int(d.attrs["msg_len"]),
                          bool(d.attrs.get("accel")))
    if codes == ["const", "addi", "crypto.digest", "yield"]:
        c, add, d, _ = ops
        if d.operands[2] is add.results[0] and {id(x) for x in add.operands} == {id(iv), id(c.results[0])}:
            return DigestLoop(v(d.operands[0]), v(d.operands[1]), d.attrs["alg"], int(d.attrs["msg_len"]),
                              bool(d.attrs.get("accel")), int(c.attrs["value"]), True)
    raise ProgramError("loop body is not the canonical crypto.digest loop")
