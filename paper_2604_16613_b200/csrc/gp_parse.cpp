// gp_parse.cpp -- native circuit text parser.
//
// Replaces parse_circuit + validate_layers (circuit.cpp:107-326): text in,
// the flat owning circuit out (gp_circuit, include/greenpeas.h), with the
// reference's grammar, rec[-k] resolution, XOR-toggled detector and
// observable sets, and its error messages ("line N: ..." for ParseError,
// "layer L: ..." for validate_layers' invalid_argument).
//
// Large texts parse in parallel on the shared host pool: the text is cut at
// line boundaries into chunks; each chunk is parsed with measurement and
// observable counts relative to its start (rec[-k] targets kept as k against
// the chunk-local count at their line), then one serial pass places the
// chunks -- measurement bases, layer boundaries at TICKs, detector ids,
// observable lists in text order -- and checks what only the global state
// can decide (a rec[-k] reaching before the first measurement, observable
// indices dense). Any error in the parallel pass re-parses the text serially,
// so the error reported is exactly the reference's first one. Layers are
// then validated in parallel (the lowest violating layer wins).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/greenpeas.h"
#include "gp_gen.h"

namespace gp {
void host_parallel_for(size_t n, const std::function<void(size_t)> &f);  // gp_api.cpp
}

namespace {

struct Fail {
    size_t line;
    std::string msg;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

struct Token {
    const char *p;
    size_t n;
    std::string str() const { return std::string(p, n); }
};

// One chunk of lines parsed relative to its start.
struct Chunk {
    const char *b = nullptr, *e = nullptr;
    size_t line0 = 0;  // lines before the chunk
    bool exact = false;  // measurement / observable state known (a serial parse): every check immediate
    // ops in text order; tick_* = op / annotation counts at each TICK (the layer closes there)
    std::vector<uint8_t> gate_kind, noise_kind;
    std::vector<uint32_t> gate_q0, gate_q1, noise_q0, noise_q1, gate_meas;
    std::vector<double> gate_flip, noise_prob;
    std::vector<uint32_t> tick_gates, tick_noise, tick_anns;
    struct Ann {
        bool obs;
        uint32_t id;            // observable index
        uint32_t meas_at;       // chunk-local measurement count at the line
        size_t line;
        std::vector<uint32_t> ks;  // rec[-k] targets, XOR-toggled (equal k = equal measurement)
    };
    std::vector<Ann> anns;
    uint32_t meas = 0, max_q = 0, obs_seen = 0;  // obs_seen: exact mode only
    bool any_q = false;
    size_t lines = 0;
    bool failed = false;
    Fail fail;

    void err(size_t line, std::string msg) {
        if (!failed) {
            failed = true;
            fail = {line, std::move(msg)};
        }
    }
};

void toggle_into(std::vector<uint32_t> &s, uint32_t t) {
    auto it = std::lower_bound(s.begin(), s.end(), t);
    if (it != s.end() && *it == t) s.erase(it);
    else s.insert(it, t);
}

// stoul semantics of parse_qubit (circuit.cpp:66-73): digits only; the value
// truncated to 32 bits; beyond 64 bits stoul throws out_of_range ("stoul").
bool parse_qubit(const Token &t, size_t line, Chunk &c, uint32_t *q) {
    uint64_t v = 0;
    bool over = false;
    for (size_t i = 0; i < t.n; i++) {
        const char ch = t.p[i];
        if (ch < '0' || ch > '9') {
            c.err(line, "expected qubit index, got '" + t.str() + "'");
            return false;
        }
        const uint64_t d = (uint64_t)(ch - '0');
        if (v > (UINT64_MAX - d) / 10) over = true;
        v = v * 10 + d;
    }
    if (over) {
        c.err(line, "stoul");
        return false;
    }
    *q = (uint32_t)v;
    return true;
}

// rec[-k] (circuit.cpp:76-92): k returned; 0 marks "reaches before the first
// measurement" (k == 0 or, in exact mode, k > the measurement count).
bool parse_rec(const Token &t, size_t line, Chunk &c, uint32_t meas_count, uint32_t *k_out) {
    auto bad = [&] {
        c.err(line, "expected rec[-k], got '" + t.str() + "'");
        return false;
    };
    if (t.n < 6 || std::strncmp(t.p, "rec[-", 5) != 0 || t.p[t.n - 1] != ']') return bad();
    uint64_t v = 0;
    bool over = false;
    for (size_t i = 5; i + 1 < t.n; i++) {
        const char ch = t.p[i];
        if (ch < '0' || ch > '9') return bad();
        const uint64_t d = (uint64_t)(ch - '0');
        if (v > (UINT64_MAX - d) / 10) over = true;
        v = v * 10 + d;
    }
    if (over) {
        c.err(line, "stoul");
        return false;
    }
    const uint32_t k = (uint32_t)v;
    if (k == 0 || (c.exact && k > meas_count)) {
        c.err(line, "record reference " + t.str() + " reaches before the first measurement");
        return false;
    }
    *k_out = k;
    return true;
}

void parse_chunk(Chunk &c) {
    std::vector<Token> tg;
    size_t line = c.line0;
    for (const char *p = c.b; p < c.e && !c.failed;) {
        const char *nl = (const char *)std::memchr(p, '\n', (size_t)(c.e - p));
        const char *le = nl ? nl : c.e;
        line++;
        c.lines++;
        const char *hash = (const char *)std::memchr(p, '#', (size_t)(le - p));
        const char *end = hash ? hash : le;
        // tokens
        tg.clear();
        for (const char *q = p; q < end;) {
            while (q < end && is_space(*q)) q++;
            if (q >= end) break;
            const char *s = q;
            while (q < end && !is_space(*q)) q++;
            tg.push_back({s, (size_t)(q - s)});
        }
        p = nl ? nl + 1 : c.e;
        if (tg.empty()) continue;
        // name and optional (argument)
        const Token &head = tg[0];
        const char *paren = (const char *)std::memchr(head.p, '(', head.n);
        std::string name;
        bool has_arg = false;
        double arg = 0;
        if (paren) {
            if (head.p[head.n - 1] != ')') {
                c.err(line, "unterminated argument in '" + head.str() + "'");
                break;
            }
            const std::string a(paren + 1, head.p + head.n - 1);
            name.assign(head.p, paren);
            char *ep = nullptr;
            arg = std::strtod(a.c_str(), &ep);
            if (ep == a.c_str() || *ep != '\0') {
                c.err(line, "bad numeric argument '" + a + "'");
                break;
            }
            has_arg = true;
        } else {
            name = head.str();
        }
        const size_t nt = tg.size() - 1;
        auto note = [&](uint32_t q) {
            c.max_q = std::max(c.max_q, q);
            c.any_q = true;
        };
        if (name == "TICK") {
            if (has_arg || nt) {
                c.err(line, "TICK takes no targets");
                break;
            }
            c.tick_gates.push_back((uint32_t)c.gate_kind.size());
            c.tick_noise.push_back((uint32_t)c.noise_kind.size());
            c.tick_anns.push_back((uint32_t)c.anns.size());
        } else if (name == "H" || name == "R") {
            if (has_arg) {
                c.err(line, name + " takes no argument");
                break;
            }
            if (!nt) {
                c.err(line, name + " needs at least one target");
                break;
            }
            for (size_t i = 1; i <= nt; i++) {
                uint32_t q;
                if (!parse_qubit(tg[i], line, c, &q)) break;
                note(q);
                c.gate_kind.push_back(name == "H" ? GP_GATE_H : GP_GATE_R);
                c.gate_q0.push_back(q);
                c.gate_q1.push_back(0);
                c.gate_meas.push_back(0xFFFFFFFFu);
                c.gate_flip.push_back(0);
            }
        } else if (name == "CX") {
            if (nt < 2 || nt % 2) {
                c.err(line, "CX needs an even number of targets");
                break;
            }
            for (size_t i = 1; i <= nt; i += 2) {
                uint32_t a, b;
                if (!parse_qubit(tg[i], line, c, &a) || !parse_qubit(tg[i + 1], line, c, &b)) break;
                if (a == b) {
                    c.err(line, "CX control equals target");
                    break;
                }
                note(a);
                note(b);
                c.gate_kind.push_back(GP_GATE_CX);
                c.gate_q0.push_back(a);
                c.gate_q1.push_back(b);
                c.gate_meas.push_back(0xFFFFFFFFu);
                c.gate_flip.push_back(0);
            }
        } else if (name == "M" || name == "MR") {
            if (!nt) {
                c.err(line, name + " needs at least one target");
                break;
            }
            for (size_t i = 1; i <= nt; i++) {
                uint32_t q;
                if (!parse_qubit(tg[i], line, c, &q)) break;
                note(q);
                c.gate_kind.push_back(name == "M" ? GP_GATE_M : GP_GATE_MR);
                c.gate_q0.push_back(q);
                c.gate_q1.push_back(0);
                c.gate_meas.push_back(c.meas++);
                c.gate_flip.push_back(has_arg ? arg : 0.0);
            }
        } else if (name == "X_ERROR" || name == "Z_ERROR" || name == "DEPOLARIZE1") {
            if (!has_arg) {
                c.err(line, name + " needs a probability argument");
                break;
            }
            const uint8_t k = name == "X_ERROR" ? GP_NOISE_X_ERROR : name == "Z_ERROR" ? GP_NOISE_Z_ERROR
                                                                                       : GP_NOISE_DEPOLARIZE1;
            for (size_t i = 1; i <= nt; i++) {
                uint32_t q;
                if (!parse_qubit(tg[i], line, c, &q)) break;
                note(q);
                c.noise_kind.push_back(k);
                c.noise_prob.push_back(arg);
                c.noise_q0.push_back(q);
                c.noise_q1.push_back(0);
            }
        } else if (name == "DEPOLARIZE2") {
            if (!has_arg) {
                c.err(line, "DEPOLARIZE2 needs a probability argument");
                break;
            }
            if (nt < 2 || nt % 2) {
                c.err(line, "DEPOLARIZE2 needs an even number of targets");
                break;
            }
            for (size_t i = 1; i <= nt; i += 2) {
                uint32_t a, b;
                if (!parse_qubit(tg[i], line, c, &a) || !parse_qubit(tg[i + 1], line, c, &b)) break;
                note(a);
                note(b);
                c.noise_kind.push_back(GP_NOISE_DEPOLARIZE2);
                c.noise_prob.push_back(arg);
                c.noise_q0.push_back(a);
                c.noise_q1.push_back(b);
            }
        } else if (name == "DETECTOR" || name == "OBSERVABLE_INCLUDE") {
            const bool obs = name == "OBSERVABLE_INCLUDE";
            Chunk::Ann an{obs, 0, c.meas, line, {}};
            if (!obs && !nt) {
                c.err(line, "DETECTOR needs at least one record target");
                break;
            }
            if (obs) {
                if (!has_arg) {
                    c.err(line, "OBSERVABLE_INCLUDE needs an index argument");
                    break;
                }
                const uint32_t id = (uint32_t)arg;
                if ((double)id != arg) {
                    c.err(line, "observable index must be an integer");
                    break;
                }
                an.id = id;
                if (c.exact) {
                    if (id > c.obs_seen) {
                        c.err(line, "observable indices must be dense");
                        break;
                    }
                    if (id == c.obs_seen) c.obs_seen++;
                }
            }
            for (size_t i = 1; i <= nt; i++) {
                uint32_t k;
                if (!parse_rec(tg[i], line, c, c.meas, &k)) break;
                toggle_into(an.ks, k);
            }
            if (c.failed) break;
            if (!obs && an.ks.empty()) {
                c.err(line, "DETECTOR measurement set cancels to empty");
                break;
            }
            c.anns.push_back(std::move(an));
        } else {
            c.err(line, "unsupported instruction '" + name + "'");
            break;
        }
    }
}

// validate_layers (circuit.cpp:254-326) over the flat circuit; layers in
// parallel, the lowest violating layer (gates before noise within a layer).
bool validate(const gp_circuit &g, std::string *msg) {
    const uint32_t L = g.layers(), n = g.num_qubits;
    const size_t k = L < 64 ? 1 : std::min<size_t>(64, L / 16);
    std::vector<std::pair<size_t, std::string>> found(k, {SIZE_MAX, {}});
    gp::host_parallel_for(k, [&](size_t part) {
        const uint32_t l0 = (uint32_t)(L * part / k), l1 = (uint32_t)(L * (part + 1) / k);
        std::vector<uint32_t> stamp(n, 0), owner(n, 0);  // qubit -> layer + 1, its gate
        for (uint32_t i = l0; i < l1; i++) {
            auto bad = [&](std::string m) {
                found[part] = {i, std::move(m)};
                return true;
            };
            bool stop = false;
            for (uint32_t x = g.gate_offsets[i]; x < g.gate_offsets[i + 1] && !stop; x++) {
                const uint32_t qs[2] = {g.gate_q0[x], g.gate_q1[x]};
                const uint32_t nq = g.gate_kind[x] == GP_GATE_CX ? 2 : 1;
                for (uint32_t j = 0; j < nq && !stop; j++) {
                    if (qs[j] >= n) stop = bad("qubit " + std::to_string(qs[j]) + " out of range");
                    else if (stamp[qs[j]] == i + 1)
                        stop = bad("qubit " + std::to_string(qs[j]) + " used by two gates in one layer");
                    else {
                        stamp[qs[j]] = i + 1;
                        owner[qs[j]] = x;
                    }
                }
                const uint8_t kd = g.gate_kind[x];
                if (!stop && (kd == GP_GATE_M || kd == GP_GATE_MR) && (g.gate_flip[x] < 0 || g.gate_flip[x] > 1))
                    stop = bad("measurement flip probability out of [0, 1]");
            }
            for (uint32_t o = g.noise_offsets[i]; o < g.noise_offsets[i + 1] && !stop; o++) {
                if (g.noise_prob[o] < 0 || g.noise_prob[o] > 1) {
                    stop = bad("noise probability out of [0, 1]");
                    break;
                }
                const bool two = g.noise_kind[o] == GP_NOISE_DEPOLARIZE2;
                const uint32_t qs[2] = {g.noise_q0[o], g.noise_q1[o]};
                for (uint32_t j = 0; j < (two ? 2u : 1u) && !stop; j++)
                    if (qs[j] >= n) stop = bad("noise qubit " + std::to_string(qs[j]) + " out of range");
                if (stop || !two) continue;
                const bool a = stamp[qs[0]] == i + 1, b = stamp[qs[1]] == i + 1;
                const uint32_t ga = owner[qs[0]];
                const bool cx_pair = a && g.gate_kind[ga] == GP_GATE_CX && g.gate_q0[ga] == qs[0] && g.gate_q1[ga] == qs[1];
                if (!(!a && !b) && !cx_pair)
                    stop = bad("DEPOLARIZE2 targets must form a CX (control, target) pair or an idle pair");
            }
            if (stop) return;
        }
    });
    for (auto &f : found)
        if (f.first != SIZE_MAX) {
            *msg = "layer " + std::to_string(f.first) + ": " + f.second;
            return false;
        }
    return true;  // (measurement order, detector and observable ids hold by construction)
}

// Places the chunks (in order) into one circuit; false (and the chunk-pass
// result abandoned) when a check needing the global state fails.
bool assemble(std::vector<Chunk> &ch, gp_circuit &g) {
    uint32_t meas_base = 0, max_q = 0;
    bool any_q = false;
    std::vector<std::vector<uint32_t>> obs;
    size_t G = 0, N = 0;
    for (const Chunk &c : ch) {
        G += c.gate_kind.size();
        N += c.noise_kind.size();
    }
    g.gate_kind.reserve(G);
    g.gate_q0.reserve(G);
    g.gate_q1.reserve(G);
    g.gate_meas.reserve(G);
    g.gate_flip.reserve(G);
    g.noise_kind.reserve(N);
    g.noise_prob.reserve(N);
    g.noise_q0.reserve(N);
    g.noise_q1.reserve(N);
    uint32_t layer = 0;  // the open layer
    size_t open_anns = 0;  // annotations placed in the open layer
    for (Chunk &c : ch) {
        size_t gi = 0, ni = 0, ai = 0;
        auto take = [&](size_t g_end, size_t n_end, size_t a_end) {
            for (; gi < g_end; gi++) {
                g.gate_kind.push_back(c.gate_kind[gi]);
                g.gate_q0.push_back(c.gate_q0[gi]);
                g.gate_q1.push_back(c.gate_q1[gi]);
                g.gate_meas.push_back(c.gate_meas[gi] == 0xFFFFFFFFu ? -1 : (int32_t)(meas_base + c.gate_meas[gi]));
                g.gate_flip.push_back(c.gate_flip[gi]);
            }
            for (; ni < n_end; ni++) {
                g.noise_kind.push_back(c.noise_kind[ni]);
                g.noise_prob.push_back(c.noise_prob[ni]);
                g.noise_q0.push_back(c.noise_q0[ni]);
                g.noise_q1.push_back(c.noise_q1[ni]);
            }
            for (; ai < a_end; ai++) {
                Chunk::Ann &a = c.anns[ai];
                std::vector<uint32_t> ms;
                ms.reserve(a.ks.size());
                const uint64_t at = (uint64_t)meas_base + a.meas_at;
                for (uint32_t k : a.ks) {
                    if (k > at) return false;  // reaches before the first measurement
                    ms.push_back((uint32_t)(at - k));
                }
                std::sort(ms.begin(), ms.end());
                if (a.obs) {
                    if (a.id > obs.size()) return false;  // not dense
                    if (a.id == obs.size()) obs.emplace_back();
                    for (uint32_t m : ms) toggle_into(obs[a.id], m);
                    g.anns.push_back({layer, true, a.id, std::move(ms)});
                } else {
                    const uint32_t id = (uint32_t)g.det_offsets.size() - 1;
                    g.det_meas.insert(g.det_meas.end(), ms.begin(), ms.end());
                    g.det_offsets.push_back((uint32_t)g.det_meas.size());
                    g.anns.push_back({layer, false, id, std::move(ms)});
                }
                open_anns++;
            }
            return true;
        };
        for (size_t t = 0; t < c.tick_gates.size(); t++) {
            if (!take(c.tick_gates[t], c.tick_noise[t], c.tick_anns[t])) return false;
            g.gate_offsets.push_back((uint32_t)g.gate_kind.size());  // TICK: the layer closes (even empty)
            g.noise_offsets.push_back((uint32_t)g.noise_kind.size());
            layer++;
            open_anns = 0;
        }
        if (!take(c.gate_kind.size(), c.noise_kind.size(), c.anns.size())) return false;
        meas_base += c.meas;
        if (c.any_q) {
            max_q = std::max(max_q, c.max_q);
            any_q = true;
        }
    }
    if (g.gate_kind.size() > g.gate_offsets.back() || g.noise_kind.size() > g.noise_offsets.back() || open_anns) {
        g.gate_offsets.push_back((uint32_t)g.gate_kind.size());  // the last layer, if not empty
        g.noise_offsets.push_back((uint32_t)g.noise_kind.size());
    }
    for (auto &o : obs) {
        g.obs_meas.insert(g.obs_meas.end(), o.begin(), o.end());
        g.obs_offsets.push_back((uint32_t)g.obs_meas.size());
    }
    g.num_qubits = any_q ? max_q + 1 : 0;
    g.num_measurements = meas_base;
    return true;
}

}  // namespace

extern "C" {

gp_circuit *gp_parse_circuit(const char *text, size_t len, char **error) {
    if (error) *error = nullptr;
    auto fail = [&](const std::string &m) -> gp_circuit * {
        if (error) {
            *error = (char *)std::malloc(m.size() + 1);
            std::memcpy(*error, m.c_str(), m.size() + 1);
        }
        return nullptr;
    };
    if (!text && len) return fail("null text");
    try {
        // chunks at line boundaries (one for small texts)
        const size_t k = len < (1u << 18) ? 1 : std::min<size_t>(256, len >> 16);
        std::vector<Chunk> ch(k);
        const char *b = text;
        for (size_t i = 0; i < k; i++) {
            const char *e = i + 1 == k ? text + len : text + len * (i + 1) / k;
            if (e < b) e = b;
            if (i + 1 < k) {  // extend to the end of the line
                const char *nl = (const char *)std::memchr(e, '\n', (size_t)(text + len - e));
                e = nl ? nl + 1 : text + len;
            }
            ch[i].b = b;
            ch[i].e = e;
            b = e;
        }
        bool serial = k == 1;
        if (!serial) {
            gp::host_parallel_for(k, [&](size_t i) { parse_chunk(ch[i]); });
            for (auto &c : ch) serial |= c.failed;
        }
        gp_circuit *g = new gp_circuit();
        if (!serial) {
            size_t line = 0;
            for (auto &c : ch) {  // (line numbers only matter for errors: all-clear here)
                c.line0 = line;
                line += c.lines;
            }
            if (!assemble(ch, *g)) {  // a check only the global state decides failed
                delete g;
                g = new gp_circuit();
                serial = true;
            }
        }
        if (serial) {  // exact: the reference's first error, or the circuit
            std::vector<Chunk> one(1);
            one[0].b = text;
            one[0].e = text + len;
            one[0].exact = true;
            parse_chunk(one[0]);
            if (one[0].failed) {
                delete g;
                return fail("line " + std::to_string(one[0].fail.line) + ": " + one[0].fail.msg);
            }
            if (!assemble(one, *g)) {  // (cannot happen in exact mode)
                delete g;
                return fail("internal: exact parse failed to assemble");
            }
        }
        std::string msg;
        if (!validate(*g, &msg)) {
            delete g;
            return fail(msg);
        }
        return g;
    } catch (const std::exception &e) {
        return fail(e.what());
    }
}

}  // extern "C"
