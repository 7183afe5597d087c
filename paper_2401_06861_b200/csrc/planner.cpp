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
//  2. Micro-op fusion inside a pass (PassBuilder):
//     - runs of dense/diagonal operators on the same bits are multiplied into
//       one pending operator per bit group; diagonal groups merge up to
//       kMaxDiagK bits;
//     - diagonal groups commute with X/CX/CCX on their control bits, so they
//       are not flushed by a permutation that only uses them as controls;
//     - a permutation P = X_t (controlled by C) that meets the same P again with
//       only diagonal work on t in between cancels: P D P = D o P is diagonal,
//       so CX.RZ.CX (ZZ rotations of TFIM/QAOA) and the CX.U1.CX halves of the
//       QFT's controlled phases become pure diagonals;
//     - other permutations, SWAP and depolarizing maps are emitted as cheap
//       dedicated micro-ops.
//  Micro-ops are kept in state-bit form and mapped to tile positions when the
//  pass is closed, so the pass caps apply to the fused (post-fusion) program.
#include "engine.hpp"
#include "knobs.hpp"

#include <algorithm>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

namespace nqe {

namespace {

uint64_t bit(int b) { return uint64_t(1) << b; }

uint64_t bitmask_of(const EOp& op, bool with_ctrl) {
    uint64_t m = 0;
    for (int j = 0; j < op.k; ++j) m |= bit(op.bits[j]);
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
        return bit(op.bits[0]);
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

// A fused operator on a small bit group (pending or emitted).
struct Group {
    int k = 0;
    int bits[kMaxDiagK];
    bool diag = true;
    std::vector<cplx> m;  // diag: 2^k; dense: 4^k row-major
    uint64_t mask() const {
        uint64_t r = 0;
        for (int j = 0; j < k; ++j) r |= bit(bits[j]);
        return r;
    }
    int index_of(int b) const {
        for (int t = 0; t < k; ++t)
            if (bits[t] == b) return t;
        return -1;
    }
};

// Local index of `sub` (its bit order) from a local index of `g`.
int sub_index(int gi, const Group& g, const int* sbits, int sk) {
    int oi = 0;
    for (int j = 0; j < sk; ++j)
        if ((gi >> g.index_of(sbits[j])) & 1) oi |= 1 << j;
    return oi;
}

void to_dense(Group& g) {
    if (!g.diag) return;
    const int d = 1 << g.k;
    std::vector<cplx> m(size_t(d) * d, cplx(0.0, 0.0));
    for (int i = 0; i < d; ++i) m[size_t(i) * d + i] = g.m[size_t(i)];
    g.m = std::move(m);
    g.diag = false;
}

// g <- op * g, op's bits a subset of g's bits.
void absorb(Group& g, const int* obits, int ok, bool odiag, const std::vector<cplx>& om) {
    const int d = 1 << g.k;
    if (odiag) {
        for (int i = 0; i < d; ++i) {
            const cplx f = om[size_t(sub_index(i, g, obits, ok))];
            if (g.diag) {
                g.m[size_t(i)] *= f;
            } else {
                for (int c = 0; c < d; ++c) g.m[size_t(i) * d + c] *= f;
            }
        }
        return;
    }
    to_dense(g);
    const int od = 1 << ok;
    uint64_t local = 0;
    for (int j = 0; j < ok; ++j) local |= bit(g.index_of(obits[j]));
    std::vector<cplx> out(size_t(d) * d, cplx(0.0, 0.0));
    for (int i = 0; i < d; ++i) {
        const int oi = sub_index(i, g, obits, ok);
        for (int ip = 0; ip < d; ++ip) {
            if ((uint64_t(i) & ~local) != (uint64_t(ip) & ~local)) continue;
            const cplx e = om[size_t(oi) * od + size_t(sub_index(ip, g, obits, ok))];
            if (e == cplx(0.0, 0.0)) continue;
            for (int c = 0; c < d; ++c) out[size_t(i) * d + c] += e * g.m[size_t(ip) * d + c];
        }
    }
    g.m = std::move(out);
}

Group group_from(const EOp& op) {
    Group g;
    g.k = op.k;
    for (int j = 0; j < op.k; ++j) g.bits[j] = op.bits[j];
    g.diag = (op.type == E_DIAG);
    g.m = op.mat;
    return g;
}

Group diag_identity_on(uint64_t mask) {
    Group g;
    g.k = 0;
    for (int b = 0; b < 64; ++b)
        if ((mask >> b) & 1) g.bits[g.k++] = b;
    g.diag = true;
    g.m.assign(size_t(1) << g.k, cplx(1.0, 0.0));
    return g;
}

bool is_identity_diag(const Group& g) {
    for (const auto& v : g.m)
        if (v != cplx(1.0, 0.0)) return false;
    return true;
}

// D o P for P = X on bit t controlled by `ctrl`, D diagonal: entry for basis
// state x is D(P x).  Result lives on D's bits plus the controls.
Group conjugate_diag(const Group& D, int t, uint64_t ctrl) {
    Group out = diag_identity_on(D.mask() | ctrl);
    const int d = 1 << out.k;
    const int tj = out.index_of(t);
    uint64_t cl = 0;
    for (int j = 0; j < out.k; ++j)
        if ((ctrl >> out.bits[j]) & 1) cl |= bit(j);
    for (int i = 0; i < d; ++i) {
        int x = i;
        if ((uint64_t(i) & cl) == cl) x ^= 1 << tj;
        out.m[size_t(i)] = D.m[size_t(sub_index(x, out, D.bits, D.k))];
    }
    return out;
}

// A micro-op in state-bit form.
struct BitOp {
    MOpType type;
    int k = 0;
    int bits[kMaxDiagK];
    uint64_t ctrl = 0;
    std::vector<cplx> m;
    bool alive = true;
    uint64_t touch() const {
        uint64_t r = ctrl;
        for (int j = 0; j < k; ++j) r |= bit(bits[j]);
        return r;
    }
};

bool stage_sched_enabled();
uint32_t coalesce_mask();

class PassBuilder {
  public:
    explicit PassBuilder(bool fuse) : fuse_(fuse) {}

    size_t microops() const { return live_ + pend_.size(); }
    size_t pool() const {
        size_t p = pool_;
        for (const auto& g : pend_) p += g.m.size();
        return p;
    }

    void add(const EOp& e) {
        if (e.type == E_NOP) return;
        if (!fuse_) {
            if (e.type == E_DENSE || e.type == E_DIAG)
                emit_group(group_from(e));
            else
                emit_direct(e);
            return;
        }
        switch (e.type) {
        case E_DENSE:
        case E_DIAG:
            add_matrix(e);
            return;
        case E_XPERM:
            add_xperm(e);
            return;
        default:
            flush_overlapping(bitmask_of(e, true), false);
            emit_direct(e);
        }
    }

    // Close the pass: map state bits to tile bits, split the micro-op program
    // into register-layout stages and encode register slots.
    // l2p: logical -> physical bit for bits outside the tile (diagonal tables
    // and controls read them from the full physical index); null = identity.
    PlannedPass finish(const std::vector<int>& q, const std::vector<int>* l2p = nullptr) {
        auto phys = [&](int b) { return l2p ? (*l2p)[size_t(b)] : b; };
        for (const auto& g : pend_) emit_group(g);
        pend_.clear();
        const int m = int(q.size());
        // register bits per thread: reg_bits_ (3 or 4), but 4 whenever an op
        // needs four register-resident bits (2-qubit superoperators)
        bool need4 = false;
        for (const auto& b : ops_)
            if (b.alive && b.k == 4 && (b.type == MOP_DENSE || b.type == MOP_DEPOL)) need4 = true;
        const int rsz = std::min(need4 ? 4 : reg_bits_, m);
        int tpos[kMaxStateBits];
        std::fill(std::begin(tpos), std::end(tpos), -1);
        for (size_t i = 0; i < q.size(); ++i) tpos[q[i]] = int(i);

        std::vector<const BitOp*> live;
        for (const auto& b : ops_)
            if (b.alive) live.push_back(&b);
        // tile bits that must be register-resident for each op
        auto need = [&](const BitOp& b) -> uint32_t {
            if (b.type == MOP_DIAG) return 0;
            const int cnt = b.type == MOP_XPERM ? 1 : b.k;
            uint32_t r = 0;
            for (int j = 0; j < cnt; ++j) {
                if (tpos[b.bits[j]] < 0) throw std::logic_error("planner: target bit outside tile");
                r |= 1u << tpos[b.bits[j]];
            }
            return r;
        };
        // fill a register set up to rsz bits with the highest free tile bits
        auto fill = [&](uint32_t r) {
            for (int t = m - 1; t >= 0 && popcount64(r) < rsz; --t) r |= 1u << t;
            return r;
        };
        // Register stages.  The pass program may be reordered where ops commute
        // (disjoint bits, or both diagonal): list scheduling over that
        // dependency DAG runs every ready op the current register set allows
        // before switching sets, and switches to the set under which the most
        // ops become runnable.  Each switch is a shared-memory relayout of the
        // whole tile, so fewer switches is less shared-memory traffic.
        const size_t L = live.size();
        std::vector<uint32_t> ndv(L);
        std::vector<uint64_t> tch(L);
        std::vector<char> isdiag(L);
        for (size_t i = 0; i < L; ++i) {
            ndv[i] = need(*live[i]);
            tch[i] = live[i]->touch();
            isdiag[i] = live[i]->type == MOP_DIAG;
        }
        std::vector<std::vector<int>> succ(L);
        std::vector<int> npred(L, 0);
        for (size_t i = 0; i < L; ++i)
            for (size_t j = i + 1; j < L; ++j)
                if ((tch[i] & tch[j]) && !(isdiag[i] && isdiag[j])) {
                    succ[i].push_back(int(j));
                    ++npred[j];
                }
        std::vector<int> order;
        std::vector<uint32_t> stage_sched;
        order.reserve(L);
        std::vector<int> np = npred;
        std::vector<char> done(L, 0);
        uint32_t cur = 0;
        bool have = false;
        // run every op runnable under register set R (need 0 or need within R),
        // on copies of the state; returns how many ran
        auto simulate = [&](uint32_t R, std::vector<int> p2, std::vector<char> d2) {
            int ran = 0;
            bool prog = true;
            while (prog) {
                prog = false;
                for (size_t i = 0; i < L; ++i) {
                    if (d2[i] || p2[i] != 0) continue;
                    if (ndv[i] != 0 && (ndv[i] & ~R) != 0) continue;
                    d2[i] = 1;
                    ++ran;
                    for (int j : succ[i]) --p2[size_t(j)];
                    prog = true;
                }
            }
            return ran;
        };
        while (order.size() < L) {
            bool prog = false;
            for (size_t i = 0; i < L; ++i) {
                if (done[i] || np[i] != 0) continue;
                if (ndv[i] != 0 && (!have || (ndv[i] & ~cur) != 0)) continue;
                done[i] = 1;
                order.push_back(int(i));
                stage_sched.push_back(cur);
                for (int j : succ[i]) --np[size_t(j)];
                prog = true;
                break;  // rescan from the lowest index: keeps program order where possible
            }
            if (prog) continue;
            // switch register sets: candidates seeded by each ready op's needs
            uint32_t best = 0;
            int best_ran = -1;
            std::vector<uint32_t> tried;
            // seed: a ready op's needs, then the needs of the following
            // unscheduled ops in program order while they fit (lookahead)
            for (size_t i = 0; i < L; ++i) {
                if (done[i] || np[i] != 0 || ndv[i] == 0) continue;
                for (int variant = 0; variant < 2; ++variant) {
                    uint32_t r = ndv[i];
                    for (size_t j = 0; j < L; ++j) {
                        if (done[j] || ndv[j] == 0 || j == i) continue;
                        if (popcount64(r | ndv[j]) <= rsz) r |= ndv[j];
                        else if (variant == 0) break;
                    }
                    r = fill(r);
                    if (std::find(tried.begin(), tried.end(), r) != tried.end()) continue;
                    tried.push_back(r);
                    const int ran = simulate(r, np, done);
                    // the first set is the load layout: on a tie, the one with
                    // fewer of the 5 lowest tile bits (the lowest physical bits)
                    // in registers, so a warp's lanes load contiguous amplitudes
                    const bool coalesce_tie = !have && ran == best_ran &&
                                              popcount64(r & 0x1Fu) < popcount64(best & 0x1Fu);
                    if (ran > best_ran || coalesce_tie) {
                        best_ran = ran;
                        best = r;
                    }
                }
            }
            if (best_ran <= 0) throw std::logic_error("planner: stage scheduling made no progress");
            if (!have) {  // ops scheduled before the first register-bound op share its layout
                for (auto& st : stage_sched) st = best;
            }
            cur = best;
            have = true;
        }
        if (!have) {
            cur = fill(0);
            for (auto& st : stage_sched) st = cur;
        }
        {
            std::vector<const BitOp*> reordered(L);
            for (size_t k = 0; k < L; ++k) reordered[k] = live[size_t(order[k])];
            live.swap(reordered);
        }
        std::vector<uint32_t> stage_of = stage_sched;
        // Program order with lookahead packing (the previous scheme) is kept
        // when it needs no more switches than the schedule.
        auto switches = [](const std::vector<uint32_t>& st) {
            int k = 0;
            for (size_t i = 1; i < st.size(); ++i) k += st[i] != st[i - 1];
            return k;
        };
        std::vector<const BitOp*> live_sched = live;
        {
            // A/B: program order, each switch packing the following ops' needs
            live.clear();
            for (const auto& b : ops_)
                if (b.alive) live.push_back(&b);
            for (size_t i = 0; i < L; ++i) ndv[i] = need(*live[i]);
            stage_of.assign(L, 0);
            uint32_t c2 = 0;
            bool h2 = false;
            for (size_t i = 0; i < L; ++i) {
                if (ndv[i] == 0 || (h2 && (ndv[i] & ~c2) == 0)) {
                    stage_of[i] = c2;
                    continue;
                }
                uint32_t r = ndv[i];
                for (size_t j = i + 1; j < L; ++j) {
                    if (popcount64(r | ndv[j]) > rsz) break;
                    r |= ndv[j];
                }
                c2 = fill(r);
                if (!h2)
                    for (size_t j = 0; j < i; ++j) stage_of[j] = c2;
                h2 = true;
                stage_of[i] = c2;
            }
            if (!h2) stage_of.assign(L, fill(0));
        }
        if (stage_sched_ && stage_sched_enabled() && switches(stage_sched) < switches(stage_of)) {
            live = live_sched;
            stage_of = stage_sched;
        }

        PlannedPass p;
        p.q = q;
        auto layout_op = [&](uint32_t r) {
            MOp op{};
            op.type = MOP_LAYOUT;
            op.k = uint8_t(rsz);
            int k = 0;
            for (int t = 0; t < m; ++t)
                if ((r >> t) & 1u) op.pos[k++] = int8_t(t);
            return op;
        };
        uint32_t lay = stage_of.empty() ? fill(0) : stage_of[0];
        // Coalescing: HBM is read and written in the first / last layout.  If
        // those hold any of the 5 lowest tile bits in registers, a warp's 32
        // lanes do not cover 32 consecutive amplitudes; then load (store) in
        // the layout of the 4 highest tile bits and relayout through shared
        // memory instead.
        const uint32_t lane_bits = m >= 9 ? coalesce_mask() : 0u;
        const uint32_t top = fill(0);
        // Always when the first stage holds 3 or 4 of the 4 lowest tile bits:
        // each lane would then load its own 128-256-byte run (the warp's
        // requests touch 16-32 lines; the L2 re-serves up to 1.75x the
        // sectors: QFT-30 pass 0).
        // (A/B: NQ_COALESCE_FULL_LOW = 1/2/3 for >= 4/3/2 of the lowest 4)
        static const int full_low = ab_knob("NQ_COALESCE_FULL_LOW", 2);
        if ((coalesce_ && (lay & lane_bits)) ||
            (full_low > 0 && m >= 9 && popcount64(lay & 0xFu) >= 5 - full_low))
            p.ops.push_back(layout_op(top));
        p.ops.push_back(layout_op(lay));
        for (size_t i = 0; i < live.size(); ++i) {
            if (stage_of[i] != lay) {
                lay = stage_of[i];
                p.ops.push_back(layout_op(lay));
            }
            const BitOp& b = *live[i];
            int slot_of_t[32];
            {
                int k = 0;
                for (int t = 0; t < m; ++t) slot_of_t[t] = ((lay >> t) & 1u) ? k++ : -1;
            }
            MOp op{};
            op.type = uint8_t(b.type);
            op.k = uint8_t(b.k);
            op.mat = uint32_t(p.pool.size());
            for (int bb = 0; bb < 64; ++bb) {
                if (!((b.ctrl >> bb) & 1)) continue;
                if (bb < kMaxStateBits && tpos[bb] >= 0)
                    op.cmask_tile |= uint32_t(1) << tpos[bb];
                else
                    op.cmask_glob |= bit(phys(bb));
            }
            if (b.type == MOP_DIAG) {
                for (int j = 0; j < b.k; ++j)
                    op.pos[j] = int8_t(tpos[b.bits[j]] >= 0 ? tpos[b.bits[j]] : -1 - phys(b.bits[j]));
                p.pool.insert(p.pool.end(), b.m.begin(), b.m.end());
            } else if (b.type == MOP_DENSE) {
                // local bit i of the stored matrix = i-th smallest slot
                int slots[4], order[4];
                for (int j = 0; j < b.k; ++j) {
                    slots[j] = slot_of_t[tpos[b.bits[j]]];
                    order[j] = j;
                }
                std::sort(order, order + b.k, [&](int x, int y) { return slots[x] < slots[y]; });
                for (int i2 = 0; i2 < b.k; ++i2) op.pos[i2] = int8_t(slots[order[i2]]);
                const int d = 1 << b.k;
                auto old_index = [&](int xn) {
                    int xo = 0;
                    for (int i2 = 0; i2 < b.k; ++i2)
                        if ((xn >> i2) & 1) xo |= 1 << order[i2];
                    return xo;
                };
                for (int r = 0; r < d; ++r)
                    for (int c = 0; c < d; ++c) p.pool.push_back(b.m[size_t(old_index(r)) * d + size_t(old_index(c))]);
            } else {
                for (int j = 0; j < b.k; ++j) op.pos[j] = int8_t(slot_of_t[tpos[b.bits[j]]]);
                if (b.type == MOP_SWAP && op.pos[0] > op.pos[1]) std::swap(op.pos[0], op.pos[1]);
                p.pool.insert(p.pool.end(), b.m.begin(), b.m.end());
            }
            p.ops.push_back(op);
        }
        if (coalesce_ && (lay & lane_bits)) p.ops.push_back(layout_op(top));
        return p;
    }

    void set_coalesce(bool c) { coalesce_ = c; }
    void set_stage_sched(bool v) { stage_sched_ = v; }
    void set_reg_bits(int r) { reg_bits_ = r; }

  private:
    void emit_group(const Group& g) {
        if (g.diag && is_identity_diag(g)) return;
        BitOp b;
        b.type = g.diag ? MOP_DIAG : MOP_DENSE;
        b.k = g.k;
        for (int j = 0; j < g.k; ++j) b.bits[j] = g.bits[j];
        b.m = g.m;
        push(std::move(b));
    }

    void emit_direct(const EOp& e) {
        BitOp b;
        b.k = e.k;
        for (int j = 0; j < e.k; ++j) b.bits[j] = e.bits[j];
        b.ctrl = e.ctrl;
        switch (e.type) {
        case E_XPERM: b.type = MOP_XPERM; break;
        case E_SWAP: b.type = MOP_SWAP; break;
        case E_DEPOL:
            b.type = MOP_DEPOL;
            b.m = e.mat;
            break;
        default: throw std::logic_error("planner: unexpected direct op");
        }
        push(std::move(b));
    }

    void push(BitOp&& b) {
        pool_ += b.m.size();
        ++live_;
        ops_.push_back(std::move(b));
    }

    // Emit pending groups overlapping `mask`; with keep_diag_ctrl, diagonal
    // groups that only overlap control bits are kept (they commute).
    void flush_overlapping(uint64_t mask, bool keep_diag_ctrl, uint64_t target = 0) {
        for (size_t i = 0; i < pend_.size();) {
            const Group& g = pend_[i];
            const bool over = (g.mask() & mask) != 0;
            const bool commutes = keep_diag_ctrl && g.diag && !(g.mask() & target);
            if (over && !commutes) {
                emit_group(g);
                pend_.erase(pend_.begin() + long(i));
            } else {
                ++i;
            }
        }
    }

    void add_matrix(const EOp& e) {
        const uint64_t emask = bitmask_of(e, false);
        std::vector<size_t> over;
        for (size_t i = 0; i < pend_.size(); ++i)
            if (pend_[i].mask() & emask) over.push_back(i);
        const bool ediag = e.type == E_DIAG;
        if (over.size() == 1) {
            Group& g = pend_[over[0]];
            if ((emask & ~g.mask()) == 0 && (!g.diag || ediag || g.k == e.k)) {
                absorb(g, e.bits, e.k, ediag, e.mat);
                return;
            }
        }
        if (ediag && !over.empty()) {
            bool all_diag = true;
            uint64_t uni = emask;
            for (size_t i : over) {
                all_diag = all_diag && pend_[i].diag;
                uni |= pend_[i].mask();
            }
            if (all_diag && popcount64(uni) <= kMaxDiagK) {
                Group mg = diag_identity_on(uni);
                for (size_t i : over) absorb(mg, pend_[i].bits, pend_[i].k, true, pend_[i].m);
                absorb(mg, e.bits, e.k, true, e.mat);
                for (size_t j = over.size(); j-- > 0;) pend_.erase(pend_.begin() + long(over[j]));
                pend_.push_back(std::move(mg));
                return;
            }
        }
        flush_overlapping(emask, false);
        pend_.push_back(group_from(e));
    }

    void add_xperm(const EOp& e) {
        const int t = e.bits[0];
        const uint64_t touched = bit(t) | e.ctrl;
        if (try_cancel(t, e.ctrl)) return;
        // diagonal groups on control bits commute with the permutation
        flush_overlapping(touched, true, bit(t));
        emit_direct(e);
    }

    // P .. (diagonal work on t) .. P  ->  conjugated diagonal, both P removed.
    bool try_cancel(int t, uint64_t ctrl) {
        const uint64_t touched = bit(t) | ctrl;
        // most recent emitted op touching t or the controls must be the same P
        long idx = -1;
        for (long i = long(ops_.size()) - 1; i >= 0; --i) {
            const BitOp& b = ops_[size_t(i)];
            if (!b.alive || !(b.touch() & touched)) continue;
            // diagonal micro-ops on control bits only commute with P
            if (b.type == MOP_DIAG && !((b.touch() >> t) & 1)) continue;
            if (b.type == MOP_XPERM && b.bits[0] == t && b.ctrl == ctrl) idx = i;
            break;
        }
        if (idx < 0) return false;
        // pending (not yet emitted) work on the controls sits between the two
        // P as well: it commutes with P only when diagonal (a dense group on
        // a control, e.g. CX(c,t) U3(c) CX(c,t), blocks the cancellation)
        for (const auto& g : pend_)
            if ((g.mask() & ctrl) && !g.diag) return false;
        // pending groups involving t must be diagonal; conjugate and merge them
        std::vector<size_t> on_t;
        uint64_t uni = 0;
        for (size_t i = 0; i < pend_.size(); ++i) {
            if (!((pend_[i].mask() >> t) & 1)) continue;
            if (!pend_[i].diag) return false;
            on_t.push_back(i);
            uni |= pend_[i].mask();
        }
        if (!on_t.empty()) {
            uni |= ctrl;
            // conjugated groups now also touch the controls: merge with any
            // pending diagonal groups there
            std::vector<size_t> merge = on_t;
            for (size_t i = 0; i < pend_.size(); ++i) {
                if (std::find(on_t.begin(), on_t.end(), i) != on_t.end()) continue;
                if (pend_[i].mask() & ctrl) {
                    if (!pend_[i].diag) return false;
                    merge.push_back(i);
                    uni |= pend_[i].mask();
                }
            }
            if (popcount64(uni) > kMaxDiagK) return false;
            Group mg = diag_identity_on(uni);
            for (size_t i : merge) {
                Group gi = pend_[i];
                if ((gi.mask() >> t) & 1) gi = conjugate_diag(gi, t, ctrl);
                absorb(mg, gi.bits, gi.k, true, gi.m);
            }
            std::sort(merge.begin(), merge.end());
            for (size_t j = merge.size(); j-- > 0;) pend_.erase(pend_.begin() + long(merge[j]));
            pend_.push_back(std::move(mg));
        }
        ops_[size_t(idx)].alive = false;
        --live_;
        return true;
    }

    bool fuse_;
    bool coalesce_ = true;
    bool stage_sched_ = true;
    int reg_bits_ = 4;
    std::vector<BitOp> ops_;
    std::vector<Group> pend_;
    size_t live_ = 0, pool_ = 0;
};

// P1..Pa  D1..Db  P1..Pa  ->  D1'..Db'  for mutually commuting X-type
// permutations P and diagonal D (D' = D o P1..Pa).  Catches CX.RZ.CX (TFIM /
// QAOA ZZ rotations), the CX.U1.CX halves of controlled phases (QFT) and, in
// Liouville space, the row+column copies of those sandwiches.
// NQ_COALESCE=1 enables the load/store relayouts.  Off by default: measured on
// B200 (random circuit n = 30, tile 11) the extra shared-memory round trips
// cost more (8.08 ms/pass) than the partially coalesced accesses (7.43 ms/pass),
// whose DRAM traffic stays exactly algorithmic (L2 merges the sectors).
bool coalesce_enabled() {
    static const bool on = ab_knob("NQ_COALESCE", 0) == 1;
    return on;
}

// Tile bits that must not be register bits of the load / store layouts
// (NQ_COALESCE_MASK, default tile bits 0-4).
uint32_t coalesce_mask() {
    static const uint32_t v = uint32_t(ab_knob("NQ_COALESCE_MASK", 0x1F));
    return v;
}

// NQ_STAGE_SCHED=0 keeps each pass program in source order (A/B).
bool stage_sched_enabled() {
    static const bool on = ab_knob("NQ_STAGE_SCHED", 1) != 0;
    return on;
}

// NQ_REGBITS=3|4 overrides PlanOptions::reg_bits (A/B measurements).
int reg_bits_env(int dflt) {
    static const int v = ab_knob("NQ_REGBITS", 0);
    return (v == 3 || v == 4) ? v : dflt;
}

bool perms_commute(const EOp& a, const EOp& b) {
    return !((a.ctrl >> b.bits[0]) & 1) && !((b.ctrl >> a.bits[0]) & 1);
}

std::vector<EOp> cancel_perm_sandwiches(const std::vector<EOp>& in) {
    std::vector<EOp> out;
    out.reserve(in.size());
    size_t i = 0;
    while (i < in.size()) {
        if (in[i].type != E_XPERM) {
            out.push_back(in[i++]);
            continue;
        }
        // leading run of commuting permutations
        size_t a = i;
        while (a < in.size() && in[a].type == E_XPERM && a - i < 4) {
            bool ok = true;
            for (size_t p = i; p < a; ++p) ok = ok && perms_commute(in[p], in[a]);
            if (!ok) break;
            ++a;
        }
        const size_t na = a - i;
        size_t d = a;
        while (d < in.size() && (in[d].type == E_DIAG || in[d].type == E_NOP)) ++d;
        bool match = d > a && d + na <= in.size();
        std::vector<bool> used(na, false);
        for (size_t t = 0; match && t < na; ++t) {
            const EOp& q = in[d + t];
            bool found = false;
            for (size_t p = 0; p < na && !found; ++p) {
                if (used[p] || q.type != E_XPERM) continue;
                if (q.bits[0] == in[i + p].bits[0] && q.ctrl == in[i + p].ctrl) {
                    used[p] = true;
                    found = true;
                }
            }
            match = found;
        }
        std::vector<EOp> conj;
        if (match) {
            for (size_t t = a; t < d && match; ++t) {
                if (in[t].type == E_NOP) {
                    conj.push_back(in[t]);
                    continue;
                }
                Group g = group_from(in[t]);
                for (size_t p = i; p < a; ++p) {
                    const int tb = in[p].bits[0];
                    if (!((g.mask() >> tb) & 1)) continue;
                    if (popcount64(g.mask() | in[p].ctrl) > kMaxDiagK) {
                        match = false;
                        break;
                    }
                    g = conjugate_diag(g, tb, in[p].ctrl);
                }
                EOp e;
                e.type = E_DIAG;
                e.k = g.k;
                for (int j = 0; j < g.k; ++j) e.bits[j] = g.bits[j];
                e.mat = g.m;
                e.src = in[t].src;
                conj.push_back(std::move(e));
            }
        }
        if (!match) {
            out.push_back(in[i++]);
            continue;
        }
        int64_t src = 0;
        for (size_t p = 0; p < na; ++p) src += in[i + p].src + in[d + p].src;
        conj.front().src += src;
        for (auto& e : conj) out.push_back(std::move(e));
        i = d + na;
    }
    return out;
}

// Global phase hoisting.  A diagonal table t acts as t[0] * (t / t[0]); the
// scalar t[0] commutes with everything, so it is multiplied into one dense
// micro-op instead (a dense op touches every amplitude exactly once).  The
// rescaled table has an exact 1 in entry 0, which the JIT turns into skipped
// complex multiplies (RZ(theta) -> diag(1, e^{i theta}) halves its FP64 work).
// Controlled micro-ops are left alone; a complex dense op is preferred as the
// carrier so real matrices keep their cheaper real form.
bool mat_is_real(const std::vector<cplx>& pool, uint32_t off, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (pool[off + i].imag() != 0.0) return false;
    return true;
}

// NQ_NORM_DENSE=0 keeps 1-qubit dense matrices as fused, 1 normalises rows
// only, 2 (default) also splits off the unit phase (A/B).
int normalise_dense_mode() {
    static const int v = ab_knob("NQ_NORM_DENSE", 2);
    return v;
}
bool normalise_dense_enabled() { return normalise_dense_mode() > 0; }

void hoist_global_phase(std::vector<PlannedPass>& passes) {
    PlannedPass* cp = nullptr;
    const MOp* carrier = nullptr;
    for (auto& p : passes) {
        for (const auto& op : p.ops) {
            if (op.type != MOP_DENSE || op.cmask_tile || op.cmask_glob) continue;
            const size_t n = size_t(1) << (2 * op.k);
            if (!carrier || (mat_is_real(cp->pool, carrier->mat, size_t(1) << (2 * carrier->k)) &&
                             !mat_is_real(p.pool, op.mat, n))) {
                carrier = &op;
                cp = &p;
            }
        }
    }
    if (!carrier) return;
    cplx phase(1.0, 0.0);
    for (auto& p : passes) {
        for (const auto& op : p.ops) {
            if (op.type != MOP_DIAG || op.cmask_tile || op.cmask_glob || op.k == 0) continue;
            const cplx f = p.pool[op.mat];
            if (f == cplx(1.0, 0.0)) continue;
            const double af = std::abs(f);
            if (!(af > 0.5 && af < 2.0)) continue;
            const cplx inv = std::conj(f) / (af * af);
            for (size_t i = 1; i < (size_t(1) << op.k); ++i) p.pool[op.mat + i] *= inv;
            p.pool[op.mat] = cplx(1.0, 0.0);
            phase *= f;
        }
    }
    // Pivot normalisation of 1-qubit dense operators (state-vector passes:
    // a Hermitian mirror pass needs every intermediate state Hermitian, so
    // density-matrix flushes with mirror passes keep their matrices).  Row 0
    // is divided by its larger entry p, so that entry is an exact 1, and the
    // other row by the same p; p joins the hoisted scalar.  The pass compiler
    // turns the exact 1 into an addition: out0 = x0 + a x1 costs 2 FP64 per
    // component instead of 4 (complex: 12 instead of 16 per amplitude pair;
    // RX / RY / H-like matrices, whose diagonal also becomes exactly +-1:
    // 4 instead of 8).  |p| >= 1/sqrt(2) for unitaries, so the scalar product
    // stays far from underflow.
    //
    // Unitaries whose normalised second row is not already +-1 on its
    // diagonal are further split as U = p * diag(1, d) * N with N having two
    // exact 1s ([[1, a], [b, 1]], or [[a, 1], [1, b]] when row 0's larger
    // entry is off the diagonal) and |d| = 1: N costs 8 FP64 per amplitude
    // pair, and the phase d follows as a 1-bit diagonal micro-op, which the
    // pass compiler accumulates per thread and folds into the next N on the
    // same register slot at run time (jit.cpp) instead of multiplying it in.
    bool mirror_flush = false;
    for (const auto& p : passes) mirror_flush = mirror_flush || (p.flags & PASS_MIRROR);
    const size_t cpi = size_t(cp - passes.data());
    const size_t coi0 = size_t(carrier - cp->ops.data());  // the carrier's index before insertions
    size_t coi = coi0;
    if (!mirror_flush && normalise_dense_enabled()) {
        for (size_t pi = 0; pi < passes.size(); ++pi) {
            PlannedPass& p = passes[pi];
            std::vector<MOp> out;
            out.reserve(p.ops.size() + 8);
            const MOp* lay = nullptr;
            for (size_t oi = 0; oi < p.ops.size(); ++oi) {
                const MOp op = p.ops[oi];
                if (pi == cpi && oi == coi0) coi = out.size();
                out.push_back(op);
                if (op.type == MOP_LAYOUT) lay = &p.ops[oi];
                if (op.type != MOP_DENSE || op.k != 1 || op.cmask_tile || op.cmask_glob || (pi == cpi && oi == coi0))
                    continue;
                cplx u[4] = {p.pool[op.mat], p.pool[op.mat + 1], p.pool[op.mat + 2], p.pool[op.mat + 3]};
                const bool diag_form = std::abs(u[0]) >= std::abs(u[1]);
                const cplx piv = diag_form ? u[0] : u[1];
                const double ap = std::abs(piv);
                if (!(ap > 0.25 && ap < 4.0)) continue;
                for (int e = 0; e < 4; ++e) u[e] = (u[e] == piv) ? cplx(1.0, 0.0) : u[e] / piv;
                phase *= piv;
                // row 1's entry under row 0's pivot: d (diag form: u11, off form: u10)
                const int de = diag_form ? 3 : 2;
                const cplx d = u[de];
                const bool unit = std::abs(std::abs(d) - 1.0) < 1e-13;
                if (normalise_dense_mode() >= 2 && unit && lay && d != cplx(1.0, 0.0) && d != cplx(-1.0, 0.0)) {
                    u[2 + (de == 3 ? 0 : 1)] /= d;
                    u[de] = cplx(1.0, 0.0);
                    MOp dg{};
                    dg.type = MOP_DIAG;
                    dg.k = 1;
                    dg.pos[0] = lay->pos[op.pos[0]];  // the dense op's register slot as a tile bit
                    dg.mat = uint32_t(p.pool.size());
                    p.pool.push_back(cplx(1.0, 0.0));
                    p.pool.push_back(d);
                    out.push_back(dg);
                }
                for (int e = 0; e < 4; ++e) p.pool[op.mat + e] = u[e];
            }
            p.ops = std::move(out);
        }
    }
    carrier = &passes[cpi].ops[coi];
    cp = &passes[cpi];
    if (phase == cplx(1.0, 0.0)) return;
    const size_t n = size_t(1) << (2 * carrier->k);
    for (size_t i = 0; i < n; ++i) cp->pool[carrier->mat + i] *= phase;
}

}  // namespace

// SWAP micro-ops at the end of a relabelling pass move no data in registers
// that anything later in the pass reads: they are folded into the store
// permutation instead (the data of tile bit i is stored where tile bit j's
// would have gone, and vice versa).  A pass left without any arithmetic (the
// bit reversal closing a QFT) then loads in a layout with its 4 highest tile
// bits in registers, so its loads are as coalesced as its stores (it had
// held the swapped low bits in registers).  The logical->physical map is
// unchanged: SWAP(a, b) o store == store with the two positions exchanged.
void absorb_trailing_swaps(PlannedPass& p) {
    if (p.ops.empty() || p.ops[0].type != MOP_LAYOUT) return;
    int last = -1;  // last op that is neither a layout nor a swap
    for (size_t i = 0; i < p.ops.size(); ++i)
        if (p.ops[i].type != MOP_LAYOUT && p.ops[i].type != MOP_SWAP) last = int(i);
    int last_layout = 0;
    for (size_t i = 0; i < p.ops.size(); ++i)
        if (p.ops[i].type == MOP_LAYOUT) last_layout = int(i);
    // with arithmetic left, only swaps after the final layout (the store
    // layout stays the one the relabelling chose)
    const int from = last < 0 ? 0 : std::max(last, last_layout);
    std::vector<std::pair<int, int>> tb;  // swapped tile bits, program order
    const MOp* lay = nullptr;
    for (size_t i = 0; i < p.ops.size(); ++i) {
        const MOp& o = p.ops[i];
        if (o.type == MOP_LAYOUT) lay = &o;
        else if (o.type == MOP_SWAP && int(i) > from && lay) tb.push_back({lay->pos[o.pos[0]], lay->pos[o.pos[1]]});
    }
    if (tb.empty()) return;
    p.lab.resize(p.q.size());
    for (size_t i = 0; i < p.lab.size(); ++i) p.lab[i] = int(i);
    for (size_t k = tb.size(); k-- > 0;) {
        std::swap(p.qst[size_t(tb[k].first)], p.qst[size_t(tb[k].second)]);
        std::swap(p.lab[size_t(tb[k].first)], p.lab[size_t(tb[k].second)]);
    }
    std::vector<MOp> keep;
    if (last < 0) {
        MOp l = p.ops[0];
        const int m = int(p.q.size());
        for (int j = 0; j < l.k; ++j) l.pos[j] = int8_t(m - l.k + j);
        keep.push_back(l);
    } else {
        for (size_t i = 0; i < p.ops.size(); ++i)
            if (!(p.ops[i].type == MOP_SWAP && int(i) > from)) keep.push_back(p.ops[i]);
    }
    p.ops.swap(keep);
}

std::vector<PlannedPass> plan_passes(const std::vector<EOp>& ops_in, const PlanOptions& opt,
                                     PlanStats* stats, std::vector<int>* map) {
    const std::vector<EOp> ops = opt.fuse ? cancel_perm_sandwiches(ops_in) : ops_in;
    const int nloc = opt.nloc;
    const int dmn = opt.dm_mirror_n;
    const bool mirror_mode = dmn > 0 && nloc > opt.tile_bits && map && int(map->size()) == opt.nbits;
    int m = std::min(opt.tile_bits, nloc);
    // A state no larger than one tile is processed whole: every bit is "low".
    // Otherwise keep >= low_bits contiguous low bits for coalescing, but always
    // leave room for one 4-bit operator among the high tile bits.
    const int lb = (nloc <= opt.tile_bits) ? m : std::max(0, std::min(opt.low_bits, m - kMaxOpK));
    if (mirror_mode && ((m - lb) & 1)) --m;  // high bits come in (column, row) pairs
    // logical partner of a density-matrix bit: column q <-> row q + n
    auto closure = [&](uint64_t mask) {
        if (!mirror_mode) return mask;
        uint64_t r = mask;
        for (int b = 0; b < 2 * dmn; ++b)
            if ((mask >> b) & 1) r |= bit(b < dmn ? b + dmn : b - dmn);
        return r;
    };
    const uint64_t all_mask = (opt.nbits >= 64) ? ~uint64_t(0) : (bit(opt.nbits) - 1);
    const uint64_t loc_mask = (nloc >= 64) ? ~uint64_t(0) : (bit(nloc) - 1);
    const bool relabel = opt.relabel && map && nloc > m && lb > 0 && int(map->size()) == opt.nbits;

    // layout: logical <-> physical bit (identity unless relabelling)
    std::vector<int> l2p(size_t(opt.nbits)), p2l(size_t(opt.nbits));
    for (int b = 0; b < opt.nbits; ++b) l2p[size_t(b)] = b;
    // a given layout is used even when it stays fixed (density matrices keep
    // an interleaved layout: qubit q's column and row bits side by side)
    if (map && int(map->size()) == opt.nbits) l2p = *map;
    for (int b = 0; b < opt.nbits; ++b) p2l[size_t(l2p[size_t(b)])] = b;
    // logical bits held by the lb low (contiguous) physical bits
    auto low_of = [&] {
        uint64_t lm = 0;
        for (int p = 0; p < lb; ++p) lm |= bit(p2l[size_t(p)]);
        return lm;
    };
    uint64_t low_mask = (lb >= 64) ? ~uint64_t(0) : low_of();

    std::vector<PlannedPass> passes;
    int64_t src_total = 0;
    for (const auto& e : ops) src_total += e.src;

    std::vector<const EOp*> remaining;
    remaining.reserve(ops.size());
    for (const auto& e : ops) {
        if (need_mask(e) & ~loc_mask) throw std::logic_error("planner: non-diagonal op on a global bit");
        remaining.push_back(&e);
    }

    struct Trial {
        PassBuilder pb;
        uint64_t qhigh = 0;
        size_t taken = 0;
        std::vector<const EOp*> next;
        bool open_pair = false;  // took a row permutation, its column copy not yet
        bool broken_pair = false;
        explicit Trial(bool fuse) : pb(fuse) {}
    };
    // One pass from `ops_list` with low bits `lowm`, the high tile bits optionally pre-seeded.
    auto build = [&](const std::vector<const EOp*>& ops_list, uint64_t seed, uint64_t lowm) {
        Trial t(opt.fuse);
        t.pb.set_coalesce(coalesce_enabled());
        t.pb.set_reg_bits(reg_bits_env(opt.reg_bits));
        t.pb.set_stage_sched(opt.stage_sched);
        t.qhigh = seed;
        uint64_t blocked = 0;
        std::vector<const EOp*> deferred;
        size_t i = 0;
        for (; i < ops_list.size(); ++i) {
            const EOp* e = ops_list[i];
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
            const uint64_t nh = t.qhigh | (closure(need_mask(*e)) & ~lowm);
            const bool fits = popcount64(nh) <= m - lb;
            const bool caps = (t.pb.microops() + 1 <= size_t(opt.max_ops_per_pass)) &&
                              (t.pb.pool() + size_t(pool_cost(*e)) <= size_t(opt.max_pool_per_pass));
            // close the pass; the rest goes to the next one (never between the
            // row and column copies of a density-matrix permutation)
            if (!caps && t.taken > 0 && !t.open_pair) break;
            if (fits) {
                if (t.open_pair && e->pair_next) t.broken_pair = true;
                t.open_pair = e->pair_next;
                t.qhigh = nh;
                t.pb.add(*e);
                ++t.taken;
            } else {
                if (t.open_pair) t.broken_pair = true;
                deferred.push_back(e);
                blocked |= touched;
                if ((blocked & all_mask) == all_mask) {
                    ++i;
                    break;
                }
            }
        }
        t.next = deferred;
        t.next.insert(t.next.end(), ops_list.begin() + long(i), ops_list.end());
        return t;
    };
    // Ops the next pass would take under low bits `lowm` (the window logic of
    // build() without building micro-ops: the relabel search's estimator).
    auto count_taken = [&](const std::vector<const EOp*>& ops_list, uint64_t lowm) {
        uint64_t qh = 0, blocked = 0;
        size_t taken = 0;
        for (const EOp* e : ops_list) {
            const uint64_t touched = bitmask_of(*e, true);
            if (touched & blocked) {
                blocked |= touched;
                if ((blocked & all_mask) == all_mask) break;
                continue;
            }
            const uint64_t nh = qh | (closure(need_mask(*e)) & ~lowm);
            if (popcount64(nh) <= m - lb) {
                qh = nh;
                ++taken;
            } else {
                blocked |= touched;
                if ((blocked & all_mask) == all_mask) break;
            }
        }
        return taken;
    };
    // Seeds: the plain in-order greedy, and the high bits most needed by the
    // next W ops (W = 24, 48, 96); keep the trial that takes the most ops.
    auto freq_seed = [&](size_t w) {
        int cnt[64] = {0};
        for (size_t i = 0; i < remaining.size() && i < w; ++i) {
            const uint64_t nm = need_mask(*remaining[i]) & ~low_mask;
            for (int b = 0; b < 64; ++b)
                if ((nm >> b) & 1) ++cnt[b];
        }
        uint64_t seed = 0;
        for (int k = 0; k < m - lb; ++k) {
            int best = -1;
            for (int b = 0; b < 64; ++b)
                if (cnt[b] > 0 && !((seed >> b) & 1) && (best < 0 || cnt[b] > cnt[best])) best = b;
            if (best < 0) break;
            seed |= bit(best);
        }
        return seed;
    };
    // Off by default: on the BASELINE workloads (random-30, QFT-30, TFIM-28,
    // VQE-28) it found no plan with fewer passes than the plain greedy.
    static const bool seeds_env = ab_knob("NQ_PLAN_SEEDS", 0) == 1;
    const bool multi_seed = seeds_env && opt.fuse && nloc > m;
    // first position at which each logical bit is a non-diagonal target in `list`
    auto next_use = [&](const std::vector<const EOp*>& list) {
        std::vector<size_t> nu(size_t(opt.nbits), SIZE_MAX);
        for (size_t i = list.size(); i-- > 0;) {
            const uint64_t nm = need_mask(*list[i]);
            for (int b = 0; b < opt.nbits; ++b)
                if ((nm >> b) & 1) nu[size_t(b)] = i;
        }
        return nu;
    };
    // home physical bit of a logical bit: identity for state vectors, the
    // interleaved (column 2q, row 2q + 1) position for density matrices
    auto home = [&](int b) { return mirror_mode ? (b < dmn ? 2 * b : 2 * (b - dmn) + 1) : b; };
    // Relabelling for density matrices works on whole qubits: the low physical
    // bit pairs hold a per-pass choice of qubits (column bit even, row bit
    // odd, as the Hermitian passes need), chosen to maximise the next pass;
    // guests leave the low pairs only to go home.
    auto relabel_pairs = [&](const std::vector<int>& q, const std::vector<const EOp*>& next) {
        const int lq = lb / 2;  // low qubit slots
        const std::vector<const EOp*> window(next.begin(), next.begin() + long(std::min<size_t>(next.size(), 128)));
        std::vector<int> units;  // tile qubits
        for (int x : q)
            if (x < dmn) units.push_back(x);
        std::vector<int> tile_pairs;
        for (int u : units) tile_pairs.push_back(l2p[size_t(u)] >> 1);
        auto in_tile = [&](int pr) { return std::find(tile_pairs.begin(), tile_pairs.end(), pr) != tile_pairs.end(); };
        std::vector<int> forced;
        for (int pr = 0; pr < lq; ++pr) {
            const int u = p2l[size_t(2 * pr)];
            if (u >= lq && !in_tile(u)) forced.push_back(u);  // a guest whose home pair is not here
        }
        auto lowmask_of = [&](const std::vector<int>& qs) {
            uint64_t mk = 0;
            for (int u : qs) mk |= closure(bit(u));
            return mk;
        };
        std::vector<int> best = forced;
        size_t best_taken = 0;
        bool have = false;
        // exhaustive over the free low slots (at most a few tile qubits)
        std::vector<int> free_units;
        for (int u : units)
            if (std::find(forced.begin(), forced.end(), u) == forced.end()) free_units.push_back(u);
        // current low qubits first: ties keep them (fewer moves)
        std::stable_sort(free_units.begin(), free_units.end(),
                         [&](int a, int b) { return (l2p[size_t(a)] >> 1) < lq && (l2p[size_t(b)] >> 1) >= lq; });
        const int need = lq - int(forced.size());
        std::vector<int> pick;
        std::function<void(size_t)> rec = [&](size_t from) {
            if (int(pick.size()) == need) {
                std::vector<int> trial = forced;
                trial.insert(trial.end(), pick.begin(), pick.end());
                const size_t tk = count_taken(window, lowmask_of(trial));
                if (!have || tk > best_taken) {
                    best = trial;
                    best_taken = tk;
                    have = true;
                }
                return;
            }
            for (size_t i = from; i < free_units.size(); ++i) {
                pick.push_back(free_units[i]);
                rec(i + 1);
                pick.pop_back();
            }
        };
        if (need > 0) rec(0);
        // placement on physical pairs of this tile
        std::vector<int> newpair(size_t(dmn), -1);
        std::vector<char> used(size_t(nloc / 2 + 1), 0);
        auto place = [&](int u, int pr) {
            newpair[size_t(u)] = pr;
            used[size_t(pr)] = 1;
        };
        auto chosen = [&](int u) { return std::find(best.begin(), best.end(), u) != best.end(); };
        for (int u : units)
            if (chosen(u) && u < lq) place(u, u);
        for (int u : units) {
            const int cur = l2p[size_t(u)] >> 1;
            if (chosen(u) && newpair[size_t(u)] < 0 && cur < lq && !used[size_t(cur)]) place(u, cur);
        }
        for (int u : units) {
            if (!chosen(u) || newpair[size_t(u)] >= 0) continue;
            for (int pr = 0; pr < lq; ++pr)
                if (!used[size_t(pr)]) {
                    place(u, pr);
                    break;
                }
        }
        for (int u : units)
            if (newpair[size_t(u)] < 0 && u >= lq && in_tile(u) && !used[size_t(u)]) place(u, u);
        for (int u : units) {
            if (newpair[size_t(u)] >= 0) continue;
            for (int pr : tile_pairs)
                if (pr >= lq && !used[size_t(pr)]) {
                    place(u, pr);
                    break;
                }
        }
        for (int u : units) {
            const int pr = newpair[size_t(u)];
            l2p[size_t(u)] = 2 * pr;
            l2p[size_t(u + dmn)] = 2 * pr + 1;
            p2l[size_t(2 * pr)] = u;
            p2l[size_t(2 * pr + 1)] = u + dmn;
        }
        low_mask = low_of();
    };
    while (!remaining.empty()) {
        Trial t = build(remaining, 0, low_mask);
        if (multi_seed) {
            for (size_t w : {size_t(24), size_t(48), size_t(96)}) {
                const uint64_t seed = freq_seed(w);
                if (!seed) continue;
                Trial c = build(remaining, seed, low_mask);
                if (c.taken > t.taken) t = std::move(c);
            }
        }
        PassBuilder& pb = t.pb;
        uint64_t qhigh = t.qhigh;
        size_t taken = t.taken;
        std::vector<const EOp*> next = std::move(t.next);
        bool pair_ok = !t.open_pair && !t.broken_pair;
        if (taken == 0 && !next.empty()) {
            // every op needs <= kMaxOpK <= m - lb high bits, so the first one always
            // fits alone; take it to guarantee progress (with its column copy)
            qhigh = closure(need_mask(*next.front())) & ~low_mask;
            const bool pair = next.front()->pair_next && next.size() > 1;
            pb.add(*next.front());
            next.erase(next.begin());
            if (pair) {
                qhigh |= closure(need_mask(*next.front())) & ~low_mask;
                pb.add(*next.front());
                next.erase(next.begin());
            }
            pair_ok = true;
        }
        // Tile bit set: low bits, required high bits, then fill.
        uint64_t qmask = low_mask | qhigh;
        std::vector<size_t> nu;
        // Last pass of a relabelling plan: when every displaced qubit fits in
        // the tile, the pass stores them home and the plan ends on the
        // identity layout (no normalising pass later; repeated circuits replan
        // to the same passes).
        bool restore = false;
        if (relabel && next.empty()) {
            uint64_t displaced = 0;
            for (int b = 0; b < nloc; ++b)
                if (l2p[size_t(b)] != home(b)) displaced |= bit(b);
            if (popcount64(qmask | displaced) <= m) {
                qmask |= displaced;
                restore = true;
            }
        }
        if (relabel && mirror_mode) {
            // fill with the qubits (column + row bit pairs) needed soonest
            nu = next_use(next);
            std::vector<int> cand;
            for (int u = 0; u < dmn; ++u)
                if (!((qmask >> u) & 1)) cand.push_back(u);
            auto unu = [&](int u) { return std::min(nu[size_t(u)], nu[size_t(u + dmn)]); };
            std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) { return unu(x) < unu(y); });
            for (int u : cand) {
                if (popcount64(qmask) + 2 > m) break;
                qmask |= closure(bit(u));
            }
        } else if (relabel) {
            // fill with the local bits the remaining ops need soonest
            nu = next_use(next);
            std::vector<int> cand;
            for (int b = 0; b < nloc; ++b)
                if (!((qmask >> b) & 1)) cand.push_back(b);
            std::stable_sort(cand.begin(), cand.end(), [&](int x, int y) { return nu[size_t(x)] < nu[size_t(y)]; });
            for (int b : cand) {
                if (popcount64(qmask) >= m) break;
                qmask |= bit(b);
            }
        } else if (mirror_mode) {
            for (int b = 0; b < dmn && popcount64(qmask) + 2 <= m; ++b) qmask |= closure(bit(b));
        } else {
            for (int b = 0; b < nloc && popcount64(qmask) < m; ++b) qmask |= bit(b);
        }
        std::vector<int> q;  // logical tile bits in ascending physical order
        for (int b = 0; b < opt.nbits; ++b)
            if ((qmask >> b) & 1) q.push_back(b);
        std::sort(q.begin(), q.end(), [&](int x, int y) { return l2p[size_t(x)] < l2p[size_t(y)]; });
        if (int(q.size()) != m) throw std::logic_error("planner: tile size mismatch");
        PlannedPass p = pb.finish(q, &l2p);
        if (p.ops.size() > 1) {
            for (size_t i = 0; i < q.size(); ++i) p.q[i] = l2p[size_t(q[i])];
            if (mirror_mode && pair_ok && closure(qmask) == qmask) {
                // physical pairs (2q, 2q+1) in the tile: mirror-closed by construction
                bool sym = true;
                for (int x : q) sym = sym && ((qmask >> (x < dmn ? x + dmn : x - dmn)) & 1);
                for (int x : q) sym = sym && (l2p[size_t(x < dmn ? x + dmn : x - dmn)] == (l2p[size_t(x)] ^ 1));
                if (sym) p.flags |= PASS_MIRROR;
            }
            if (restore) {
                for (int x : q) {
                    l2p[size_t(x)] = home(x);
                    p2l[size_t(home(x))] = x;
                }
                low_mask = low_of();
            } else if (relabel && mirror_mode && !next.empty()) {
                relabel_pairs(q, next);
            } else if (relabel && !next.empty()) {
                // Choose the tile qubits that the low physical bits hold after this
                // pass: greedily, the set under which the next pass takes the most ops.
                // A guest (a qubit whose home is a high bit, held by a low bit)
                // only leaves the low bits to go home, so it stays when its home
                // bit is not in this tile: at most 2 * lb qubits are ever displaced.
                // the next pass is judged on a bounded window of the remaining ops
                const std::vector<const EOp*> window(next.begin(),
                                                     next.begin() + long(std::min<size_t>(next.size(), 128)));
                uint64_t chosen = 0;
                {
                    std::vector<int> tile_phys;
                    for (int x : q) tile_phys.push_back(l2p[size_t(x)]);
                    for (int pbit = 0; pbit < lb; ++pbit) {
                        const int g = p2l[size_t(pbit)];
                        if (g >= lb && std::find(tile_phys.begin(), tile_phys.end(), g) == tile_phys.end())
                            chosen |= bit(g);
                    }
                }
                for (int slot = popcount64(chosen); slot < lb; ++slot) {
                    int best = -1;
                    size_t best_taken = 0;
                    std::vector<int> order(q);
                    // current low qubits first (ties keep them: fewer moves)
                    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
                        return ((low_mask >> x) & 1) > ((low_mask >> y) & 1);
                    });
                    for (int c : order) {
                        if ((chosen >> c) & 1) continue;
                        uint64_t trial = chosen | bit(c);
                        // complete the trial set with the soonest-needed remaining tile qubits
                        std::vector<int> rest;
                        for (int x : q)
                            if (!((trial >> x) & 1)) rest.push_back(x);
                        std::stable_sort(rest.begin(), rest.end(),
                                         [&](int x, int y) { return nu[size_t(x)] < nu[size_t(y)]; });
                        for (int x : rest) {
                            if (popcount64(trial) >= lb) break;
                            trial |= bit(x);
                        }
                        const size_t tk = count_taken(window, trial);
                        if (best < 0 || tk > best_taken) {
                            best = c;
                            best_taken = tk;
                        }
                    }
                    chosen |= bit(best);
                }
                // New layout, any permutation of this tile's physical bits: the
                // chosen qubits take the low bits, and every qubit whose home bit
                // is free goes home (fewer displaced qubits to restore later).
                std::vector<int> phys_set;
                for (int x : q) phys_set.push_back(l2p[size_t(x)]);
                std::vector<int> newpos(size_t(opt.nbits), -1);
                std::vector<char> used(size_t(opt.nbits), 0);
                auto place = [&](int x, int pos) {
                    newpos[size_t(x)] = pos;
                    used[size_t(pos)] = 1;
                };
                // 1) chosen qubits.  Those held in registers by the pass's last
                //    layout take the highest low bits, so the warp's lanes (its
                //    thread bits, ordered by store position) span the lowest
                //    physical bits and the stores stay fully coalesced; within
                //    each group: home if home is free, then stay, then any.
                //    (A pass with a single layout stores through an extra
                //    relayout whose register bits the pass compiler picks.)
                uint64_t regq = 0;
                int nlay = 0;
                for (const auto& o : p.ops) nlay += o.type == MOP_LAYOUT;
                for (auto it = p.ops.rbegin(); it != p.ops.rend() && nlay > 1; ++it)
                    if (it->type == MOP_LAYOUT) {
                        for (int j = 0; j < it->k; ++j) regq |= bit(q[size_t(it->pos[j])]);
                        break;
                    }
                int nthr = 0;
                for (int x : q) nthr += ((chosen >> x) & 1) && !((regq >> x) & 1);
                for (int grp = 0; grp < 2; ++grp) {
                    const int lo = grp == 0 ? 0 : nthr, hi = grp == 0 ? nthr : lb;
                    auto member = [&](int x) { return ((chosen >> x) & 1) && (((regq >> x) & 1) != 0) == (grp == 1); };
                    for (int x : q)
                        if (member(x) && x >= lo && x < hi && !used[size_t(x)]) place(x, x);
                    for (int x : q)
                        if (member(x) && newpos[size_t(x)] < 0 && l2p[size_t(x)] >= lo && l2p[size_t(x)] < hi &&
                            !used[size_t(l2p[size_t(x)])])
                            place(x, l2p[size_t(x)]);
                    for (int x : q) {
                        if (!member(x) || newpos[size_t(x)] >= 0) continue;
                        for (int pbit = lo; pbit < hi; ++pbit)
                            if (!used[size_t(pbit)]) {
                                place(x, pbit);
                                break;
                            }
                    }
                }
                // 2) the others: home when it is a free high bit of this tile, else any free high bit
                auto in_tile = [&](int pos) { return std::find(phys_set.begin(), phys_set.end(), pos) != phys_set.end(); };
                for (int x : q)
                    if (newpos[size_t(x)] < 0 && x >= lb && in_tile(x) && !used[size_t(x)]) place(x, x);
                for (int x : q) {
                    if (newpos[size_t(x)] >= 0) continue;
                    for (int pos : phys_set)
                        if (pos >= lb && !used[size_t(pos)]) {
                            place(x, pos);
                            break;
                        }
                }
                for (int x : q) {
                    l2p[size_t(x)] = newpos[size_t(x)];
                    p2l[size_t(newpos[size_t(x)])] = x;
                }
                low_mask = low_of();
            }
            p.qst.resize(q.size());
            for (size_t i = 0; i < q.size(); ++i) p.qst[i] = l2p[size_t(q[i])];
            if (relabel && !(p.flags & PASS_MIRROR)) absorb_trailing_swaps(p);
            passes.push_back(std::move(p));
        }
        remaining.swap(next);
    }
    if (opt.fuse) hoist_global_phase(passes);
    if (stats) {
        stats->passes = int64_t(passes.size());
        stats->microops = 0;
        for (const auto& p : passes) stats->microops += int64_t(p.ops.size());
        stats->source_ops = src_total;
    }
    if (relabel) *map = l2p;
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
        for (size_t i = 0; i < p.q.size(); ++i) {
            h.q[i] = int8_t(p.q[i]);
            h.qst[i] = int8_t(p.qst.empty() ? p.q[i] : p.qst[i]);
            h.lab[i] = int8_t(p.lab.empty() ? int(i) : p.lab[i]);
        }
        h.flags = p.flags;
        int nr = 0;
        uint64_t qm = 0;
        for (int b : p.q) qm |= bit(b);
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
