// Gate-fusion planner (subsystem 1 of the north star; no counterpart in the
// reference, which applies one full-state sweep per GateOp:
// proj/src/statevector.cpp:198-222, proj/src/densitymatrix.cpp:114-167).
//
// Two levels:
//  1. Pass windows.  Ops are scanned in order; an op joins the current pass
//     when the bits it needs inside the tile (non-diagonal targets) fit in the
//     pass's m-bit tile set Q and none of the bits it touches is "blocked" by an
//     earlier deferred op.  Deferred ops block every bit they touch, so an op
//     is only ever moved ahead of ops it is disjoint from (they commute).
//  2. Micro-op fusion inside a pass.  Runs of dense/diagonal operators on the
//     same bits are multiplied into one pending operator per bit group;
//     diagonal operators may merge into one diagonal on up to 4 bits;
//     permutations (X/CX/CCX/SWAP) and depolarizing maps flush the groups
//     they touch and are emitted as cheap dedicated micro-ops.
#include "engine.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>

namespace nqe {

namespace {

uint64_t bitmask_of(const EOp& op, bool with_ctrl) {
    uint64_t m = 0;
    for (int j = 0; j < op.k; ++j) m |= uint64_t(1) << op.bits[j];
    if (with_ctrl) m |= op.ctrl;
    return m;
}

// Bits that must be tile bits for this op to execute inside a pass.
uint64_t need_mask(const EOp& op) {
    switch (op.type) {
    case E_DENSE:
    case E_DEPOL:
    case E_SWAP:
        return bitmask_of(op, false);
    case E_XPERM:
        return uint64_t(1) << op.bits[0];
    default:
        return 0;  // diagonal and no-op need no tile bits
    }
}

int pool_cost(const EOp& op) {
    switch (op.type) {
    case E_DENSE: return 1 << (2 * op.k);
    case E_DIAG: return 1 << op.k;
    case E_DEPOL: return 2;
    default: return 0;
    }
}

int popcount64(uint64_t x) { return __builtin_popcountll(x); }

// A pending (not yet emitted) fused operator on a small bit group.
struct Pending {
    int k = 0;
    int bits[4];
    bool diag = true;
    std::vector<cplx> m;  // diag: 2^k; dense: 4^k row-major
    uint64_t mask() const {
        uint64_t r = 0;
        for (int j = 0; j < k; ++j) r |= uint64_t(1) << bits[j];
        return r;
    }
};

// Local index (in group g's bit order) -> local index of `op` restricted to op's bits.
int sub_index(int gi, const Pending& g, const EOp& op) {
    int oi = 0;
    for (int j = 0; j < op.k; ++j) {
        int pos = -1;
        for (int t = 0; t < g.k; ++t)
            if (g.bits[t] == op.bits[j]) pos = t;
        if ((gi >> pos) & 1) oi |= 1 << j;
    }
    return oi;
}

void to_dense(Pending& g) {
    if (!g.diag) return;
    const int d = 1 << g.k;
    std::vector<cplx> m(size_t(d) * d, cplx(0.0, 0.0));
    for (int i = 0; i < d; ++i) m[size_t(i) * d + i] = g.m[size_t(i)];
    g.m = std::move(m);
    g.diag = false;
}

// g <- op * g, op's bits a subset of g's bits.
void absorb(Pending& g, const EOp& op) {
    const int d = 1 << g.k;
    if (op.type == E_DIAG) {
        if (g.diag) {
            for (int i = 0; i < d; ++i) g.m[size_t(i)] *= op.mat[size_t(sub_index(i, g, op))];
        } else {
            for (int i = 0; i < d; ++i) {
                const cplx f = op.mat[size_t(sub_index(i, g, op))];
                for (int c = 0; c < d; ++c) g.m[size_t(i) * d + c] *= f;
            }
        }
        return;
    }
    // dense op
    to_dense(g);
    const int od = 1 << op.k;
    uint64_t opmask_local = 0;  // op bits in g-local positions
    for (int j = 0; j < op.k; ++j)
        for (int t = 0; t < g.k; ++t)
            if (g.bits[t] == op.bits[j]) opmask_local |= uint64_t(1) << t;
    std::vector<cplx> out(size_t(d) * d, cplx(0.0, 0.0));
    for (int i = 0; i < d; ++i) {
        const int oi = sub_index(i, g, op);
        for (int ip = 0; ip < d; ++ip) {
            if ((uint64_t(i) & ~opmask_local) != (uint64_t(ip) & ~opmask_local)) continue;
            const cplx e = op.mat[size_t(oi) * od + size_t(sub_index(ip, g, op))];
            if (e == cplx(0.0, 0.0)) continue;
            for (int c = 0; c < d; ++c) out[size_t(i) * d + c] += e * g.m[size_t(ip) * d + c];
        }
    }
    g.m = std::move(out);
}

Pending pending_from(const EOp& op) {
    Pending g;
    g.k = op.k;
    for (int j = 0; j < op.k; ++j) g.bits[j] = op.bits[j];
    g.diag = (op.type == E_DIAG);
    g.m = op.mat;
    return g;
}

// Merge diagonal groups (all diagonal) and a diagonal op into one group.
Pending merge_diag(const std::vector<Pending*>& groups, const EOp& op) {
    Pending out;
    out.k = 0;
    auto add_bit = [&](int b) {
        for (int t = 0; t < out.k; ++t)
            if (out.bits[t] == b) return;
        out.bits[out.k++] = b;
    };
    for (auto* g : groups)
        for (int j = 0; j < g->k; ++j) add_bit(g->bits[j]);
    for (int j = 0; j < op.k; ++j) add_bit(op.bits[j]);
    const int d = 1 << out.k;
    out.diag = true;
    out.m.assign(size_t(d), cplx(1.0, 0.0));
    for (auto* g : groups) {
        EOp as_op;
        as_op.type = E_DIAG;
        as_op.k = g->k;
        for (int j = 0; j < g->k; ++j) as_op.bits[j] = g->bits[j];
        as_op.mat = g->m;
        absorb(out, as_op);
    }
    absorb(out, op);
    return out;
}

bool is_identity_diag(const Pending& g) {
    for (const auto& v : g.m)
        if (v != cplx(1.0, 0.0)) return false;
    return true;
}

class PassBuilder {
  public:
    PassBuilder(const std::vector<int>& q, int nloc) : q_(q) {
        std::fill(std::begin(tpos_), std::end(tpos_), -1);
        for (size_t i = 0; i < q.size(); ++i) tpos_[q[i]] = int(i);
        (void)nloc;
    }

    void emit_pending(const Pending& g) {
        if (g.diag && is_identity_diag(g)) return;
        MOp op{};
        op.k = uint8_t(g.k);
        op.mat = uint32_t(pass_.pool.size());
        if (g.diag) {
            op.type = MOP_DIAG;
            for (int j = 0; j < g.k; ++j) {
                op.pos[j] = int8_t(tpos_[g.bits[j]]);
                op.gq[j] = uint8_t(g.bits[j]);
            }
        } else {
            op.type = MOP_DENSE;
            for (int j = 0; j < g.k; ++j) {
                if (tpos_[g.bits[j]] < 0) throw std::logic_error("planner: dense bit outside tile");
                op.pos[j] = int8_t(tpos_[g.bits[j]]);
            }
        }
        pass_.pool.insert(pass_.pool.end(), g.m.begin(), g.m.end());
        pass_.ops.push_back(op);
    }

    void emit_direct(const EOp& e) {
        MOp op{};
        op.k = uint8_t(e.k);
        op.mat = uint32_t(pass_.pool.size());
        switch (e.type) {
        case E_XPERM:
            op.type = MOP_XPERM;
            op.pos[0] = int8_t(tpos_[e.bits[0]]);
            for (int b = 0; b < 64; ++b) {
                if (!((e.ctrl >> b) & 1)) continue;
                if (b < kMaxStateBits && tpos_[b] >= 0)
                    op.cmask_tile |= uint32_t(1) << tpos_[b];
                else
                    op.cmask_glob |= uint64_t(1) << b;
            }
            break;
        case E_SWAP:
            op.type = MOP_SWAP;
            op.pos[0] = int8_t(tpos_[e.bits[0]]);
            op.pos[1] = int8_t(tpos_[e.bits[1]]);
            break;
        case E_DEPOL:
            op.type = MOP_DEPOL;
            for (int j = 0; j < e.k; ++j) op.pos[j] = int8_t(tpos_[e.bits[j]]);
            pass_.pool.push_back(e.mat[0]);
            pass_.pool.push_back(e.mat[1]);
            break;
        case E_DENSE:
        case E_DIAG:
            emit_pending(pending_from(e));
            return;
        default:
            return;
        }
        for (int j = 0; j < e.k && e.type != E_XPERM; ++j)
            if (op.pos[j] < 0) throw std::logic_error("planner: target bit outside tile");
        if (op.pos[0] < 0) throw std::logic_error("planner: target bit outside tile");
        pass_.ops.push_back(op);
    }

    void flush_overlapping(uint64_t mask) {
        for (size_t i = 0; i < pend_.size();) {
            if (pend_[i].mask() & mask) {
                emit_pending(pend_[i]);
                pend_.erase(pend_.begin() + long(i));
            } else {
                ++i;
            }
        }
    }

    void add(const EOp& e, bool fuse) {
        if (e.type == E_NOP) return;
        if (!fuse) {
            emit_direct(e);
            return;
        }
        const uint64_t touched = bitmask_of(e, true);
        if ((e.type == E_DENSE || e.type == E_DIAG) && e.ctrl == 0) {
            std::vector<size_t> over;
            for (size_t i = 0; i < pend_.size(); ++i)
                if (pend_[i].mask() & touched) over.push_back(i);
            const uint64_t emask = bitmask_of(e, false);
            if (over.size() == 1) {
                Pending& g = pend_[over[0]];
                const bool subset = (emask & ~g.mask()) == 0;
                if (subset) {
                    if (!g.diag || e.type == E_DIAG) {
                        absorb(g, e);
                        return;
                    }
                    if (g.k == e.k) {  // diag group on exactly these bits, dense op
                        absorb(g, e);
                        return;
                    }
                }
            }
            if (e.type == E_DIAG && !over.empty()) {
                bool all_diag = true;
                uint64_t uni = emask;
                for (size_t i : over) {
                    all_diag = all_diag && pend_[i].diag;
                    uni |= pend_[i].mask();
                }
                if (all_diag && popcount64(uni) <= kMaxOpK) {
                    std::vector<Pending*> gs;
                    for (size_t i : over) gs.push_back(&pend_[i]);
                    Pending merged = merge_diag(gs, e);
                    for (size_t j = over.size(); j-- > 0;) pend_.erase(pend_.begin() + long(over[j]));
                    pend_.push_back(std::move(merged));
                    return;
                }
            }
            flush_overlapping(touched);
            pend_.push_back(pending_from(e));
            return;
        }
        flush_overlapping(touched);
        emit_direct(e);
    }

    PlannedPass finish() {
        for (const auto& g : pend_) emit_pending(g);
        pend_.clear();
        pass_.q = q_;
        return std::move(pass_);
    }

  private:
    std::vector<int> q_;
    int tpos_[kMaxStateBits];
    std::vector<Pending> pend_;
    PlannedPass pass_;
};

}  // namespace

std::vector<PlannedPass> plan_passes(const std::vector<EOp>& ops, const PlanOptions& opt,
                                     PlanStats* stats) {
    const int nloc = opt.nloc;
    const int m = std::min(opt.tile_bits, nloc);
    // A state no larger than one tile is processed whole: every bit is "low".
    // Otherwise keep >= low_bits contiguous low bits for coalescing, but always
    // leave room for one 4-bit operator among the high tile bits.
    const int lb = (nloc <= opt.tile_bits) ? m : std::max(0, std::min(opt.low_bits, m - kMaxOpK));
    const uint64_t low_mask = (lb >= 64) ? ~uint64_t(0) : ((uint64_t(1) << lb) - 1);
    const uint64_t all_mask =
        (opt.nbits >= 64) ? ~uint64_t(0) : ((uint64_t(1) << opt.nbits) - 1);
    const uint64_t loc_mask = (nloc >= 64) ? ~uint64_t(0) : ((uint64_t(1) << nloc) - 1);

    std::vector<PlannedPass> passes;
    int64_t src_total = 0;
    for (const auto& e : ops) src_total += e.src;

    std::vector<const EOp*> remaining;
    remaining.reserve(ops.size());
    for (const auto& e : ops) {
        if (need_mask(e) & ~loc_mask) throw std::logic_error("planner: non-diagonal op on a global bit");
        remaining.push_back(&e);
    }

    while (!remaining.empty()) {
        uint64_t qhigh = 0;  // required tile bits >= lb
        uint64_t blocked = 0;
        int nops = 0, pool = 0;
        std::vector<const EOp*> in_pass, deferred;
        size_t i = 0;
        for (; i < remaining.size(); ++i) {
            const EOp* e = remaining[i];
            const uint64_t touched = bitmask_of(*e, true);
            if (touched & blocked) {
                deferred.push_back(e);
                blocked |= touched;
                if ((blocked & all_mask) == all_mask) {
                    ++i;
                    break;
                }
                continue;
            }
            const uint64_t nh = qhigh | (need_mask(*e) & ~low_mask);
            const bool fits = popcount64(nh) <= m - lb;
            const bool caps = (nops + 1 <= opt.max_ops_per_pass) &&
                              (pool + pool_cost(*e) <= opt.max_pool_per_pass);
            if (!caps) break;  // close the pass here; the rest goes to the next pass
            if (fits) {
                qhigh = nh;
                in_pass.push_back(e);
                ++nops;
                pool += pool_cost(*e);
            } else {
                deferred.push_back(e);
                blocked |= touched;
                if ((blocked & all_mask) == all_mask) {
                    ++i;
                    break;
                }
            }
        }
        std::vector<const EOp*> next = deferred;
        next.insert(next.end(), remaining.begin() + long(i), remaining.end());
        if (in_pass.empty()) {
            if (next.size() == remaining.size() && !next.empty()) {
                // A single op must always fit (k <= 4 <= m - lb is guaranteed by callers);
                // take it alone to guarantee progress.
                in_pass.push_back(next.front());
                qhigh = need_mask(*next.front()) & ~low_mask;
                next.erase(next.begin());
            }
        }
        // Tile bit set: low bits, required high bits, then fill upward.
        uint64_t qmask = low_mask | qhigh;
        for (int b = 0; b < nloc && popcount64(qmask) < m; ++b) qmask |= uint64_t(1) << b;
        std::vector<int> q;
        for (int b = 0; b < nloc; ++b)
            if ((qmask >> b) & 1) q.push_back(b);
        if (int(q.size()) != m) throw std::logic_error("planner: tile size mismatch");

        PassBuilder pb(q, nloc);
        for (const EOp* e : in_pass) pb.add(*e, opt.fuse);
        PlannedPass p = pb.finish();
        if (!p.ops.empty()) passes.push_back(std::move(p));
        remaining.swap(next);
    }
    if (stats) {
        stats->passes = int64_t(passes.size());
        stats->microops = 0;
        for (const auto& p : passes) stats->microops += int64_t(p.ops.size());
        stats->source_ops = src_total;
    }
    return passes;
}

std::vector<unsigned char> serialize_passes(const std::vector<PlannedPass>& passes, int nloc,
                                            std::vector<size_t>* offsets) {
    std::vector<unsigned char> buf;
    if (offsets) offsets->clear();
    for (const auto& p : passes) {
        PassHdr h;
        std::memset(&h, 0, sizeof(h));
        h.m = int32_t(p.q.size());
        h.nops = int32_t(p.ops.size());
        h.nloc = nloc;
        h.ntiles = int64_t(1) << (nloc - h.m);
        for (size_t i = 0; i < p.q.size(); ++i) h.q[i] = int8_t(p.q[i]);
        int nr = 0;
        uint64_t qm = 0;
        for (int b : p.q) qm |= uint64_t(1) << b;
        for (int b = 0; b < nloc; ++b)
            if (!((qm >> b) & 1)) h.rest[nr++] = int8_t(b);
        h.nrest = nr;
        h.op_off = uint32_t(sizeof(PassHdr));
        h.pool_off = uint32_t(sizeof(PassHdr) + p.ops.size() * sizeof(MOp));
        h.pool_off = (h.pool_off + 15u) & ~15u;
        h.pool_n = uint32_t(p.pool.size());
        h.bytes = uint32_t(h.pool_off + p.pool.size() * sizeof(cplx));
        h.bytes = (h.bytes + 15u) & ~15u;
        const size_t at = buf.size();
        if (offsets) offsets->push_back(at);
        buf.resize(at + h.bytes, 0);
        std::memcpy(buf.data() + at, &h, sizeof(h));
        if (!p.ops.empty())
            std::memcpy(buf.data() + at + h.op_off, p.ops.data(), p.ops.size() * sizeof(MOp));
        if (!p.pool.empty())
            std::memcpy(buf.data() + at + h.pool_off, p.pool.data(), p.pool.size() * sizeof(cplx));
    }
    return buf;
}

}  // namespace nqe
