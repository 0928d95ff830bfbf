// sf_plan.hpp -- host-only exchange planning (no CUDA calls).
//
// One refresh phase of exchanger::refresh_worker (exchange.hpp:107-119) for the
// grid components a process owns: block-to-block copies between local
// components, bc_face fills of physical faces, and the messages to and from
// components owned by other processes (ranks).  Messages to one peer are
// concatenated in a fixed order so that sender and receiver agree without any
// handshake:
//   sender   : for field f (ascending), for axis a, sides 0 then 1
//   receiver : for field f (ascending), for axis a, sides 1 then 0
// A component's side-s face lands in the peer's side-(1-s) ghosts, so the k-th
// message of a pair matches on both ends even when both faces of a periodic
// axis face the same peer (2 ranks along that axis).  Two components that are
// neighbours share exactly one axis, so the per-axis order suffices when
// several axes go in one phase (the fused loop's divu face exchange).
#pragma once

#include <array>
#include <map>
#include <vector>

namespace sfb {

struct plan_box {
  int field = 0;
  int axis = 0, side = 0;
  int blk = 0;       // local block index (the block read for sends / copies / bc, written for recvs)
  int dst_blk = 0;   // copies: local destination block
  long long lo[3]{}, dims[3]{}, dlo[3]{};
  long long count = 0;
};

struct phase_plan {
  std::vector<plan_box> copies;                   // local block -> local block
  std::vector<plan_box> bcs;                      // physical faces (axis phase only)
  std::map<int, std::vector<plan_box>> sends;     // peer rank -> boxes in posting order
  std::map<int, std::vector<plan_box>> recvs;     // peer rank -> ghost boxes in posting order
};

// decomposition access the planner needs (global worker ids)
template <class Dec>
phase_plan build_phase_plan(const Dec& dec, const std::vector<int>& gid, const std::vector<int>& lid,
                            const std::vector<int>& owner, unsigned mask, const std::vector<int>& axes,
                            bool widen, bool exchange_only, bool skip_self) {
  phase_plan P;
  const long long g = dec.ghost;
  for (int b = 0; b < (int)gid.size(); ++b) {
    const int gw = gid[b];
    const auto dims = dec.dims(gw);
    for (int f = 0; f < 32; ++f) {
      if (!(mask & (1u << f))) continue;
      for (int a : axes) {
        auto send_box = [&](int side) {
          plan_box p;
          p.field = f;
          p.axis = a;
          p.side = side;
          p.blk = b;
          for (int t = 0; t < 3; ++t) {
            if (t == a) {
              p.lo[t] = side == 0 ? 0 : dims[t] - g;
              p.dims[t] = g;
            } else if (t < a && widen) {
              p.lo[t] = -g;
              p.dims[t] = dims[t] + 2 * g;
            } else {
              p.lo[t] = 0;
              p.dims[t] = dims[t];
            }
          }
          p.count = p.dims[0] * p.dims[1] * p.dims[2];
          return p;
        };
        for (int side = 0; side < 2; ++side) {
          const int nb = dec.neighbor(gw, a, side);
          if (nb < 0) {
            if (exchange_only || !widen) continue;
            plan_box p;
            p.field = f;
            p.axis = a;
            p.side = side;
            p.blk = b;
            for (int t = 0; t < 3; ++t) {
              if (t == a) {
                p.lo[t] = 0;
                p.dims[t] = 1;
              } else if (t < a) {
                p.lo[t] = -g;
                p.dims[t] = dims[t] + 2 * g;
              } else {
                p.lo[t] = 0;
                p.dims[t] = dims[t];
              }
            }
            p.count = p.dims[0] * p.dims[1] * p.dims[2];
            P.bcs.push_back(p);
            continue;
          }
          if (g == 0) continue;
          if (skip_self && nb == gw) continue;
          plan_box p = send_box(side);
          if (lid[nb] >= 0) {
            const auto nbd = dec.dims(nb);
            p.dst_blk = lid[nb];
            for (int t = 0; t < 3; ++t) p.dlo[t] = p.lo[t];
            p.dlo[a] = side == 0 ? nbd[a] : -g;
            P.copies.push_back(p);
          } else {
            P.sends[owner[nb]].push_back(p);
          }
        }
        for (int side = 1; side >= 0; --side) {
          const int nb = dec.neighbor(gw, a, side);
          if (nb < 0 || g == 0 || lid[nb] >= 0) continue;
          if (skip_self && nb == gw) continue;
          plan_box p = send_box(side);  // tangential extents match the sender's
          p.lo[a] = side == 0 ? -g : dims[a];
          P.recvs[owner[nb]].push_back(p);
        }
      }
    }
  }
  return P;
}

// The temporal pass's exchange as direct stores (no phases): for each of the
// 26 directions d in {-1,0,1}^3 \ 0 whose neighbour exists (every non-zero
// axis leads through a processor face, periodic wraps included, and the
// neighbour is another component), the g owned layers along each non-zero
// axis of d (all owned cells along the zero axes) go straight into that
// neighbour's ghost shell: d = -1 -> its high ghosts [m, m+g), d = +1 -> its
// low ghosts [-g, 0), d = 0 -> the same local index (the neighbour shares the
// coordinate). For every ghost cell whose out-of-range axes all lead through
// processor faces this is the value the three exchange-only axis phases
// (exchange.hpp:107-119, slabs widened over earlier axes) deliver, since that
// chain ends at the same diagonal neighbour's owned cell.
struct direct_box {
  int peer = -1;
  int d[3]{};
  long long lo[3]{}, dims[3]{}, dlo[3]{};
  long long count = 0;
};

template <class Dec>
std::vector<direct_box> build_direct_plan(const Dec& dec, int w) {
  std::vector<direct_box> out;
  const long long g = dec.ghost;
  const auto c = dec.coords_of(w);
  const auto n = dec.dims(w);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int d[3] = {dx, dy, dz};
        if (!dx && !dy && !dz) continue;
        std::array<int, 3> cp = c;
        bool ok = true;
        for (int a = 0; a < 3 && ok; ++a) {
          if (!d[a]) continue;
          cp[a] += d[a];
          if (cp[a] < 0 || cp[a] >= dec.pg[a]) {
            if (!dec.periodic[a]) ok = false;
            cp[a] = (cp[a] + dec.pg[a]) % dec.pg[a];
          }
        }
        if (!ok || g == 0) continue;
        const int peer = dec.id_of(cp);
        if (peer == w) continue;
        const auto m = dec.dims(peer);
        direct_box b;
        b.peer = peer;
        for (int a = 0; a < 3; ++a) {
          b.d[a] = d[a];
          if (d[a] < 0) {
            b.lo[a] = 0;
            b.dims[a] = g;
            b.dlo[a] = m[a];
          } else if (d[a] > 0) {
            b.lo[a] = n[a] - g;
            b.dims[a] = g;
            b.dlo[a] = -g;
          } else {
            b.lo[a] = 0;
            b.dims[a] = n[a];
            b.dlo[a] = 0;
          }
        }
        b.count = b.dims[0] * b.dims[1] * b.dims[2];
        out.push_back(b);
      }
  return out;
}

}  // namespace sfb
