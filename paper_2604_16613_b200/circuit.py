"""Flat circuit model + the reference circuit grammar (host side, never timed).

`Circuit` holds the structure-of-arrays layout of include/greenpeas.h
(gp_circuit_view), which mirrors demc::Circuit
(/root/reference/proj/core/include/demc/circuit.hpp:33-97).

`parse_circuit` / `serialize_circuit` follow circuit.cpp:107-252 / 328-388
(TICK-delimited layers, rec[-k] resolution, XOR-toggled detector and
observable sets, validate_layers on parse) so fixture text from the reference
loads unchanged and generated circuits can be handed to the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GATE_H, GATE_CX, GATE_R, GATE_M, GATE_MR = range(5)
NOISE_X, NOISE_Z, NOISE_DEP1, NOISE_DEP2 = range(4)
_NOISE_NAMES = {"X_ERROR": NOISE_X, "Z_ERROR": NOISE_Z, "DEPOLARIZE1": NOISE_DEP1, "DEPOLARIZE2": NOISE_DEP2}
_NOISE_TEXT = {v: k for k, v in _NOISE_NAMES.items()}


class ParseError(ValueError):
    """Malformed circuit text (circuit.hpp:27-31); carries the 1-based line."""

    def __init__(self, line: int, msg: str):
        super().__init__(f"line {line}: {msg}")
        self.line = line


@dataclass
class Circuit:
    num_qubits: int
    num_measurements: int
    gate_offsets: np.ndarray  # u32 [L+1]
    gate_kind: np.ndarray  # u8
    gate_q0: np.ndarray  # u32
    gate_q1: np.ndarray  # u32
    gate_meas: np.ndarray  # i32
    gate_flip: np.ndarray  # f64
    noise_offsets: np.ndarray  # u32 [L+1]
    noise_kind: np.ndarray  # u8
    noise_prob: np.ndarray  # f64
    noise_q0: np.ndarray  # u32
    noise_q1: np.ndarray  # u32
    det_offsets: np.ndarray  # u32 [D+1]
    det_meas: np.ndarray  # u32
    obs_offsets: np.ndarray  # u32 [O+1]
    obs_meas: np.ndarray  # u32
    # (layer, is_observable, id, measurements) in declaration order; only
    # used to place annotations when serializing.
    annotations: list = field(default_factory=list)

    @property
    def num_layers(self) -> int:
        return len(self.gate_offsets) - 1

    @property
    def num_detectors(self) -> int:
        return len(self.det_offsets) - 1

    @property
    def num_observables(self) -> int:
        return len(self.obs_offsets) - 1

    def detectors(self):
        return [self.det_meas[self.det_offsets[d]:self.det_offsets[d + 1]] for d in range(self.num_detectors)]

    def observables(self):
        return [self.obs_meas[self.obs_offsets[o]:self.obs_offsets[o + 1]] for o in range(self.num_observables)]

    def same_as(self, other: "Circuit") -> bool:
        """Structural equality of everything compile_circuit reads."""
        names = ["gate_offsets", "gate_kind", "gate_q0", "gate_meas", "noise_offsets", "noise_kind",
                 "noise_q0", "det_offsets", "det_meas", "obs_offsets", "obs_meas"]
        if (self.num_qubits, self.num_measurements) != (other.num_qubits, other.num_measurements):
            return False
        for n in names:
            if not np.array_equal(getattr(self, n), getattr(other, n)):
                return False
        cx = self.gate_kind == GATE_CX
        if not np.array_equal(self.gate_q1[cx], other.gate_q1[cx]):
            return False
        m = (self.gate_kind == GATE_M) | (self.gate_kind == GATE_MR)
        if not np.array_equal(self.gate_flip[m], other.gate_flip[m]):
            return False
        d2 = self.noise_kind == NOISE_DEP2
        return bool(np.array_equal(self.noise_prob, other.noise_prob)
                    and np.array_equal(self.noise_q1[d2], other.noise_q1[d2]))


class _Builder:
    def __init__(self):
        self.g_off, self.g_kind, self.g_q0, self.g_q1, self.g_meas, self.g_flip = [0], [], [], [], [], []
        self.n_off, self.n_kind, self.n_prob, self.n_q0, self.n_q1 = [0], [], [], [], []
        self.dets: list[list[int]] = []
        self.obs: list[list[int]] = []
        self.anns = []
        self.cur_gates = self.cur_noise = self.cur_anns = 0

    def flush(self):
        self.g_off.append(len(self.g_kind))
        self.n_off.append(len(self.n_kind))
        self.cur_gates = self.cur_noise = self.cur_anns = 0

    def finish(self, num_qubits: int, num_meas: int) -> Circuit:
        det_off = np.zeros(len(self.dets) + 1, np.uint32)
        det_off[1:] = np.cumsum([len(d) for d in self.dets]) if self.dets else []
        obs_off = np.zeros(len(self.obs) + 1, np.uint32)
        obs_off[1:] = np.cumsum([len(o) for o in self.obs]) if self.obs else []
        return Circuit(
            num_qubits=num_qubits, num_measurements=num_meas,
            gate_offsets=np.array(self.g_off, np.uint32), gate_kind=np.array(self.g_kind, np.uint8),
            gate_q0=np.array(self.g_q0, np.uint32), gate_q1=np.array(self.g_q1, np.uint32),
            gate_meas=np.array(self.g_meas, np.int32), gate_flip=np.array(self.g_flip, np.float64),
            noise_offsets=np.array(self.n_off, np.uint32), noise_kind=np.array(self.n_kind, np.uint8),
            noise_prob=np.array(self.n_prob, np.float64), noise_q0=np.array(self.n_q0, np.uint32),
            noise_q1=np.array(self.n_q1, np.uint32), det_offsets=det_off,
            det_meas=np.array([m for d in self.dets for m in d], np.uint32), obs_offsets=obs_off,
            obs_meas=np.array([m for o in self.obs for m in o], np.uint32), annotations=self.anns)


def _toggle(s: list[int], t: int) -> None:
    import bisect
    i = bisect.bisect_left(s, t)
    if i < len(s) and s[i] == t:
        s.pop(i)
    else:
        s.insert(i, t)


def _qubit(tok: str, line: int) -> int:
    if not tok.isdigit():
        raise ParseError(line, f"expected qubit index, got '{tok}'")
    return int(tok)


def _rec(tok: str, meas_count: int, line: int) -> int:
    if not (tok.startswith("rec[-") and tok.endswith("]")) or not tok[5:-1].isdigit():
        raise ParseError(line, f"expected rec[-k], got '{tok}'")
    k = int(tok[5:-1])
    if k == 0 or k > meas_count:
        raise ParseError(line, f"record reference {tok} reaches before the first measurement")
    return meas_count - k


def parse_circuit(text: str) -> Circuit:
    """circuit.cpp:107-252 (grammar) + validate_layers (circuit.cpp:254-326)."""
    b = _Builder()
    meas_count = 0
    max_q = -1
    for line_no, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0]
        toks = line.split()
        if not toks:
            continue
        head, targets = toks[0], toks[1:]
        arg = None
        if "(" in head:
            if not head.endswith(")"):
                raise ParseError(line_no, f"unterminated argument in '{head}'")
            name, a = head[:head.index("(")], head[head.index("(") + 1:-1]
            try:
                arg = float(a)
            except ValueError:
                raise ParseError(line_no, f"bad numeric argument '{a}'") from None
        else:
            name = head
        if name == "TICK":
            if arg is not None or targets:
                raise ParseError(line_no, "TICK takes no targets")
            b.flush()
        elif name in ("H", "R"):
            if arg is not None:
                raise ParseError(line_no, f"{name} takes no argument")
            if not targets:
                raise ParseError(line_no, f"{name} needs at least one target")
            for t in targets:
                q = _qubit(t, line_no)
                max_q = max(max_q, q)
                b.g_kind.append(GATE_H if name == "H" else GATE_R)
                b.g_q0.append(q), b.g_q1.append(0), b.g_meas.append(-1), b.g_flip.append(0.0)
                b.cur_gates += 1
        elif name == "CX":
            if len(targets) < 2 or len(targets) % 2:
                raise ParseError(line_no, "CX needs an even number of targets")
            for i in range(0, len(targets), 2):
                a, c = _qubit(targets[i], line_no), _qubit(targets[i + 1], line_no)
                if a == c:
                    raise ParseError(line_no, "CX control equals target")
                max_q = max(max_q, a, c)
                b.g_kind.append(GATE_CX)
                b.g_q0.append(a), b.g_q1.append(c), b.g_meas.append(-1), b.g_flip.append(0.0)
                b.cur_gates += 1
        elif name in ("M", "MR"):
            if not targets:
                raise ParseError(line_no, f"{name} needs at least one target")
            for t in targets:
                q = _qubit(t, line_no)
                max_q = max(max_q, q)
                b.g_kind.append(GATE_M if name == "M" else GATE_MR)
                b.g_q0.append(q), b.g_q1.append(0), b.g_meas.append(meas_count)
                b.g_flip.append(arg if arg is not None else 0.0)
                meas_count += 1
                b.cur_gates += 1
        elif name in ("X_ERROR", "Z_ERROR", "DEPOLARIZE1"):
            if arg is None:
                raise ParseError(line_no, f"{name} needs a probability argument")
            for t in targets:
                q = _qubit(t, line_no)
                max_q = max(max_q, q)
                b.n_kind.append(_NOISE_NAMES[name]), b.n_prob.append(arg), b.n_q0.append(q), b.n_q1.append(0)
                b.cur_noise += 1
        elif name == "DEPOLARIZE2":
            if arg is None:
                raise ParseError(line_no, "DEPOLARIZE2 needs a probability argument")
            if len(targets) < 2 or len(targets) % 2:
                raise ParseError(line_no, "DEPOLARIZE2 needs an even number of targets")
            for i in range(0, len(targets), 2):
                a, c = _qubit(targets[i], line_no), _qubit(targets[i + 1], line_no)
                max_q = max(max_q, a, c)
                b.n_kind.append(NOISE_DEP2), b.n_prob.append(arg), b.n_q0.append(a), b.n_q1.append(c)
                b.cur_noise += 1
        elif name == "DETECTOR":
            if not targets:
                raise ParseError(line_no, "DETECTOR needs at least one record target")
            s: list[int] = []
            for t in targets:
                _toggle(s, _rec(t, meas_count, line_no))
            if not s:
                raise ParseError(line_no, "DETECTOR measurement set cancels to empty")
            b.anns.append((len(b.g_off) - 1, False, len(b.dets), list(s)))
            b.dets.append(s)
            b.cur_anns += 1
        elif name == "OBSERVABLE_INCLUDE":
            if arg is None:
                raise ParseError(line_no, "OBSERVABLE_INCLUDE needs an index argument")
            oid = int(arg)
            if oid != arg:
                raise ParseError(line_no, "observable index must be an integer")
            if oid > len(b.obs):
                raise ParseError(line_no, "observable indices must be dense")
            if oid == len(b.obs):
                b.obs.append([])
            s = []
            for t in targets:
                _toggle(s, _rec(t, meas_count, line_no))
            for mm in s:
                _toggle(b.obs[oid], mm)
            b.anns.append((len(b.g_off) - 1, True, oid, list(s)))
            b.cur_anns += 1
        else:
            raise ParseError(line_no, f"unsupported instruction '{name}'")
    if b.cur_gates or b.cur_noise or b.cur_anns:
        b.flush()
    c = b.finish(max_q + 1, meas_count)
    v = validate_layers(c)
    if v is not None:
        raise ValueError(f"layer {v[0]}: {v[1]}")
    return c


def validate_layers(c: Circuit):
    """circuit.cpp:254-326: returns (layer, message) of the first violation or None."""
    nxt = 0
    big = 2**64 - 1
    for i in range(c.num_layers):
        owner = {}
        for g in range(c.gate_offsets[i], c.gate_offsets[i + 1]):
            k = int(c.gate_kind[g])
            qs = [int(c.gate_q0[g])] + ([int(c.gate_q1[g])] if k == GATE_CX else [])
            for q in qs:
                if q >= c.num_qubits:
                    return i, f"qubit {q} out of range"
                if q in owner:
                    return i, f"qubit {q} used by two gates in one layer"
                owner[q] = g
            if k in (GATE_M, GATE_MR):
                if int(c.gate_meas[g]) != nxt:
                    return i, "measurement indices out of order"
                nxt += 1
                if not 0 <= c.gate_flip[g] <= 1:
                    return i, "measurement flip probability out of [0, 1]"
        for o in range(c.noise_offsets[i], c.noise_offsets[i + 1]):
            if not 0 <= c.noise_prob[o] <= 1:
                return i, "noise probability out of [0, 1]"
            k = int(c.noise_kind[o])
            qs = [int(c.noise_q0[o])] + ([int(c.noise_q1[o])] if k == NOISE_DEP2 else [])
            for q in qs:
                if q >= c.num_qubits:
                    return i, f"noise qubit {q} out of range"
            if k == NOISE_DEP2:
                a, bq = owner.get(qs[0]), owner.get(qs[1])
                idle = a is None and bq is None
                cx = (a is not None and c.gate_kind[a] == GATE_CX and c.gate_q0[a] == qs[0]
                      and c.gate_q1[a] == qs[1])
                if not idle and not cx:
                    return i, "DEPOLARIZE2 targets must form a CX (control, target) pair or an idle pair"
    if nxt != c.num_measurements:
        return big, "measurement count mismatch"
    for d, ms in enumerate(c.detectors()):
        if len(ms) == 0:
            return big, f"detector {d} has empty measurement set"
        if np.any(ms >= c.num_measurements):
            return big, f"detector {d} references missing measurement"
    return None


def _fmt(x: float) -> str:
    """Round-trip text for circuit arguments (parsed back by strtod / float)."""
    return repr(float(x))


def serialize_circuit(c: Circuit) -> str:
    """circuit.cpp:328-388: gates, noise, then the layer's annotations."""
    out = []
    meas = 0
    anns = sorted(c.annotations, key=lambda a: a[0]) if c.annotations else _default_annotations(c)
    ai = 0
    for i in range(c.num_layers):
        if i:
            out.append("TICK")
        for g in range(c.gate_offsets[i], c.gate_offsets[i + 1]):
            k = int(c.gate_kind[g])
            q = int(c.gate_q0[g])
            if k == GATE_H:
                out.append(f"H {q}")
            elif k == GATE_R:
                out.append(f"R {q}")
            elif k == GATE_CX:
                out.append(f"CX {q} {int(c.gate_q1[g])}")
            else:
                name = "M" if k == GATE_M else "MR"
                f = float(c.gate_flip[g])
                out.append(f"{name}({_fmt(f)}) {q}" if f != 0 else f"{name} {q}")
                meas += 1
        for o in range(c.noise_offsets[i], c.noise_offsets[i + 1]):
            k = int(c.noise_kind[o])
            tail = f" {int(c.noise_q1[o])}" if k == NOISE_DEP2 else ""
            out.append(f"{_NOISE_TEXT[k]}({_fmt(float(c.noise_prob[o]))}) {int(c.noise_q0[o])}{tail}")
        while ai < len(anns) and anns[ai][0] == i:
            _, is_obs, aid, ms = anns[ai]
            head = f"OBSERVABLE_INCLUDE({aid})" if is_obs else "DETECTOR"
            out.append(" ".join([head] + [f"rec[-{meas - m}]" for m in ms]))
            ai += 1
    return "".join(s + "\n" for s in out)


def _default_annotations(c: Circuit):
    """Place each detector / observable at the layer of its last measurement."""
    layer_of = np.zeros(max(c.num_measurements, 1), np.int64)
    for i in range(c.num_layers):
        sel = c.gate_meas[c.gate_offsets[i]:c.gate_offsets[i + 1]]
        layer_of[sel[sel >= 0]] = i
    anns = []
    for d, ms in enumerate(c.detectors()):
        anns.append((int(layer_of[int(ms.max())]), False, d, [int(m) for m in ms]))
    last = c.num_layers - 1
    for o, ms in enumerate(c.observables()):
        anns.append((last, True, o, [int(m) for m in ms]))
    anns.sort(key=lambda a: (a[0], a[1], a[2]))
    return anns


def merge_prob(a: float, b: float) -> float:
    """dem.hpp:28-30 (Python floats are IEEE doubles; no FMA)."""
    return a * (1 - b) + b * (1 - a)


def is_close(a: float, b: float, rel: float = 1e-12) -> bool:
    return math.isclose(a, b, rel_tol=rel, abs_tol=0.0) or a == b
