// Host orchestration of the device pipeline and the C ABI (include/sdns_cuda.h).
//
// One sdns_ctx is one rank: its layout (build_layout), wavenumber geometry
// (computed in-register by the kernels, mesh.cpp:23-89), the twiddle table,
// the transpose work buffers and the communicator(s). It replaces the
// reference's DistributedFFT + WavenumberMesh + RhsWorkspace
// (fft.cpp:15-57, mesh.cpp:23-72, navier_stokes.hpp:32-41).
//
// Device layout: spectral components are (s0, s1, pitch)
// complex with pitch = round_up(s2, 8); real components are (r0, r1, r2)
// doubles. Slab work buffers:
//   wa  "x layout"  (n, np, pitch) x 6 comps  -- send buffer of the inverse
//        transpose / receive buffer of the forward one
//   wb  "y layout"  [peer][x_l][y_l][pitch] x 6 comps -- the receive layout,
//        read directly by the y pass (no unpack pass); aliases wa at p = 1.
#include <algorithm>
#include <array>
#include <initializer_list>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <mutex>

#include "host.h"
#include "kernels.cuh"

using namespace sdns_host;
using sdns_dev::ColGeom;
using sdns_dev::RowMap;
using sdns_dev::SpecGeom;
using sdns_dev::WaveGeom;
using sdns_dev::XfArgs;

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SDNS_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SDNS_INTERNAL_ERROR;
  } catch (...) {
    g_last_error = "unknown error";
    return SDNS_INTERNAL_ERROR;
  }
}

int ilog2(long long v) {
  int s = 0;
  while ((1LL << s) < v) ++s;
  return s;
}

bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

// Device layout of one rank: spectral components are x planes
// of `prow` = s1 + 1 rows (one pad row) of `pitch` = round_up(s2, 8) complex.
sdns_dev_layout dev_layout(const sdns_config& cfg, const sdns_layout& lo) {
  sdns_dev_layout d{};
  d.pitch = static_cast<int>((lo.spec_shape[2] + 7) / 8 * 8);
  d.prow = static_cast<int>(lo.spec_shape[1]) + 1;
  d.np = cfg.decomp == SDNS_PENCIL ? cfg.n / cfg.p1 : cfg.n / cfg.p;
  d.spec_cs = lo.spec_shape[0] * d.prow * d.pitch;
  d.real_cs = lo.real_shape[0] * lo.real_shape[1] * lo.real_shape[2];
  return d;
}

// Slab transpose plan: per field and peer q, the x planes [q np, (q+1) np)
// of the x layout (wa) are one contiguous block; received blocks land back to
// back as [q][x_l][y_l] planes -- the receive layout the y pass reads
// directly (no pack/unpack pass; replaces fft.cpp:89-95 and :116-122).
// Entries: (peer, offset in source, offset in destination, complex count);
// inverse: wa -> wb, forward: wb -> wa.
std::vector<std::array<long long, 4>> exchange_plan(const sdns_config& cfg, const sdns_layout& lo,
                                                     bool inverse_dir, int nfields) {
  const sdns_dev_layout d = dev_layout(cfg, lo);
  const long long blk = static_cast<long long>(d.np) * d.prow * d.pitch;
  std::vector<std::array<long long, 4>> plan;
  for (int f = 0; f < nfields; ++f)
    for (int q = 0; q < cfg.p; ++q) {
      const long long off = f * d.spec_cs + q * blk;
      plan.push_back({q, off, off, blk});
    }
  (void)inverse_dir;  // the slab plan is symmetric
  return plan;
}

}  // namespace

struct sdns_field;

struct sdns_ctx {
  sdns_config cfg{};
  sdns_ctx_options opt{};
  sdns_layout lo{};
  int device = 0;
  std::shared_ptr<Comm> world;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double2* tw = nullptr;
  double2* wa = nullptr;
  double2* wb = nullptr;
  // p = 1 slab: P1 output / P2 input in the chunk-major layout
  // [kz chunk][y][x][8] (5 fields of cs_x): P1 writes every tile as one
  // contiguous 64 KB block instead of 512 rows 2 MB apart, P2 reads it back
  // with 64 KB strides.
  double2* wx = nullptr;
  long long cs_x = 0;
  // p = 1 with wx: P2 .. P5a work in the chunked layout [x][kz chunk][y][8]
  // (x planes padded to an odd multiple of 128 B): P2 and P4 move
  // contiguous 64 KB tiles, the z pass stages each half-row as one
  // tensor-map box of pitch/8 chunks
  bool zchunk = false;
  // n = 1024 on one rank: the work fields stay in wa (no memory for wx) in a
  // chunk-major layout [kz chunk][x][y][8] from P1 to P5a (see cm_y)
  bool cmx = false;
  long long spec_cs = 0;   // complex elements per spectral component (padded)
  int prow = 0;            // rows per x plane incl. one pad row (s1 + 1)
  long long real_cs = 0;   // doubles per real component
  int pitch = 0;
  int np = 0;              // slab block n/p; pencil n/p1 (= x_l = y_l2)
  double norm = 1.0;
  // Pencil (p = p1 x p2, fft.cpp:130-227): row group (same coord1, size p2,
  // trades kz for y) and column group (same coord2, size p1, trades y for
  // x). wc: row-send/receive layout [q][x_l][y_l][pitch]; wd: z lines as p2
  // kz segments [q][x_l][y_l][pitch_q].
  bool pencil = false;
  std::shared_ptr<Comm> row, col;
  // Host wait for the context stream through the world communicator's
  // watchdog (Comm::wait); a failure also abandons the pencil sub-groups.
  void wait() {
    try {
      world->wait(stream);
    } catch (const Error& e) {
      for (auto* g : {&row, &col})
        if (*g) (*g)->abandon(e.code, e.what());
      throw;
    }
  }
  // Releases whatever has been allocated, also when sdns_ctx_create throws
  // part way (an OOM on a work buffer, a failed peer mapping).
  ~sdns_ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    if (cstream) {
      cudaStreamSynchronize(cstream);
      for (auto& e : xev)
        if (e) cudaEventDestroy(e);
      cudaStreamDestroy(cstream);
    }
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (peer_grp && !peer_wb.empty()) peer_grp->unmap_peers(peer_wb);
    if (peer_grp && !peer_wa.empty()) peer_grp->unmap_peers(peer_wa);
    if (row && !peer_wd.empty()) row->unmap_peers(peer_wd);
    if (row && !peer_wc.empty()) row->unmap_peers(peer_wc);
    for (void* p : {static_cast<void*>(d_seg), static_cast<void*>(d_seg_row),
                    static_cast<void*>(tw), static_cast<void*>(wc), static_cast<void*>(wd),
                    static_cast<void*>(wx), static_cast<void*>(d_partial),
                    static_cast<void*>(d_fpartial), static_cast<void*>(d_dts),
                    static_cast<void*>(d_fout), static_cast<void*>(d_out),
                    static_cast<void*>(d_flag)})
      if (p) cudaFree(p);
    if (wb && wb != wa) cudaFree(wb);
    if (wa) cudaFree(wa);
    if (h_out) cudaFreeHost(h_out);
    if (h_fout) cudaFreeHost(h_fout);
    if (h_flag) cudaFreeHost(h_flag);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
  double2* wc = nullptr;
  double2* wd = nullptr;
  long long cs_c = 0, cs_d = 0;
  int yl = 0;  // real y block n/p2
  std::vector<long long> seg_base;
  std::vector<int> seg_pitch, seg_k0, seg_b;
  double* d_partial = nullptr;
  double* d_out = nullptr;
  // sampled diagnostics fused into the last stage of a step (sdns_advance):
  // valid for field fused_u while the sample hook runs
  double* d_fpartial = nullptr;
  double* d_fout = nullptr;
  const sdns_field* fused_u = nullptr;
  // pinned copy of d_fout fetched with the sampled step's finite flag (one
  // host synchronisation per sampled step instead of two); valid while
  // fused_on_host
  double* h_fout = nullptr;
  bool fused_on_host = false;
  double* d_dts = nullptr;  // dt-dependent scalars of captured steps
  // slab p > 1: transposes on their own stream, overlapped with the FFT
  // passes of the other field groups (events order the two streams)
  cudaStream_t cstream = nullptr;
  cudaEvent_t xev[12] = {};
  // slab p > 1, peer-direct transposes: P1 stores into every
  // rank's wb and P4 into every rank's wa; d_seg = [inverse (wb) | forward
  // (wa)] element offsets of each destination block from the own buffer.
  bool peer = false;
  std::vector<void*> peer_wa, peer_wb;
  long long* d_seg = nullptr;
  Comm* peer_grp = nullptr;  // the group the peer-direct transposes run over
  int peer_n = 0;            // its size
  // pencil row group (p2 > 1), peer-direct kz-block transposes: P2 stores its
  // y-block q rows into member q's wd (d_seg_row), the z pass stores kz
  // segment q into member q's wc (zmo_row, an output RowMap).
  bool peer_row = false;
  // true while the last thing on the stream was a peer-direct RHS: its
  // closing barrier already orders the next fused stores after every
  // rank's reads of the work buffers; any other entry point clears it and
  // the next RHS opens with a barrier (stores into a peer's buffers must
  // wait for whatever that peer still has queued on them).
  bool peer_fresh = false;
  std::vector<void*> peer_wd, peer_wc;
  long long* d_seg_row = nullptr;
  RowMap zmo_row;
  double* h_out = nullptr;  // pinned
  int* d_flag = nullptr;
  int* h_flag = nullptr;    // pinned
  int shells = 0;
  int64_t dev_bytes = 0;
  // Optional per-pass CUDA-event timing (bench.py's live roofline). Events
  // are created when timing is enabled, never inside a step.
  bool timing = false;
  // captured steps (see step_impl): [0] plain, [1] with fused diagnostics
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    const sdns_state* st = nullptr;
    int post_project = -1;
  };
  StepGraph graphs[2];
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_tag;
  size_t ev_used = 0;

  int tick(int tag) {
    if (!timing) return -1;
    if (ev_used + 2 > ev.size()) return -1;
    const int i = static_cast<int>(ev_used);
    ev_used += 2;
    ev_tag[static_cast<size_t>(i)] = tag;
    cudaEventRecord(ev[static_cast<size_t>(i)], stream);
    return i;
  }
  void tock(int i) {
    if (i >= 0) cudaEventRecord(ev[static_cast<size_t>(i) + 1], stream);
  }

  SpecGeom sgeom() const {
    SpecGeom g;
    g.n = cfg.n;
    g.s0 = static_cast<int>(lo.spec_shape[0]);
    g.s1 = static_cast<int>(lo.spec_shape[1]);
    g.s2 = static_cast<int>(lo.spec_shape[2]);
    g.o0 = static_cast<int>(lo.spec_offset[0]);
    g.o1 = static_cast<int>(lo.spec_offset[1]);
    g.o2 = static_cast<int>(lo.spec_offset[2]);
    g.pitch = pitch;
    g.prow = prow;
    g.cs = spec_cs;
    return g;
  }
  long long plane() const { return static_cast<long long>(prow) * pitch; }
  // x pass over the x layout: rows = local y, positions = x (full axis)
  ColGeom xgeom() const {
    ColGeom g;
    g.rs = pitch;
    g.ps0 = plane();
    g.ps1 = 0;
    g.pb_shift = 30;
    g.nrows = np;
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    g.row_off = static_cast<int>(lo.spec_offset[1]);
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = prow;
    g.single = opt.p1_single > 0 || (opt.p1_single == 0 && cfg.n >= 1024);
    return g;
  }
  ColGeom xl_out() const {  // x-pass view of wx: rows = y, positions = x
    ColGeom g = xgeom();
    const long long n = cfg.n;
    g.rs = n * 8;
    g.ps0 = 8;
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[1]) * n * 8;
    g.mrows = static_cast<int>(lo.spec_shape[1]);
    return g;
  }
  ColGeom xl_in() const {  // y-pass view of wx: rows = x, positions = y
    ColGeom g;
    const long long n = cfg.n;
    g.rs = 8;
    g.ps0 = n * 8;
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[1]) * n * 8;
    g.nrows = static_cast<int>(n);
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = static_cast<int>(n);
    return g;
  }
  // chunked work layout (zchunk): x-plane stride and the pass views
  long long xpl() const { return static_cast<long long>(pitch / 8) * lo.spec_shape[1] * 8 + 8; }
  ColGeom yc_geom() const {  // y passes: rows = x, positions = y
    ColGeom g;
    g.rs = xpl();
    g.ps0 = 8;
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[1]) * 8;
    g.nrows = static_cast<int>(lo.spec_shape[0]);
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = static_cast<int>(lo.spec_shape[0]);
    return g;
  }
  ColGeom yc_geom_fwd() const {  // forward y pass, pruned like ygeom_fwd
    ColGeom g = yc_geom();
    if (!cfg.dealias) return g;
    const int K = keep_k();
    const int kzk = std::max(0, std::min(g.n2, K + 1 - static_cast<int>(lo.spec_offset[2])));
    g.n2 = kzk;
    g.pitch = std::max(8, (kzk + 7) / 8 * 8);
    g.keep_k = K;
    return g;
  }
  ColGeom xc_geom_fwd() const {  // forward x pass input: rows = y, positions = x
    ColGeom g = xgeom_fwd();     // (enumeration and pruning of the x layout)
    g.rs = 8;
    g.ps0 = xpl();
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[1]) * 8;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = static_cast<int>(lo.spec_shape[1]);
    return g;
  }
  // In-place chunk-major work layout [kz chunk][x][y][8] (cmx): element
  // (x, y, kz) of a field at (kz >> 3) * n * s1 * 8 + x * s1 * 8 + y * 8 +
  // (kz & 7). The y passes (P2, P4: 14.3 C of traffic per RHS) then move
  // contiguous tiles in place; the x passes see positions s1 * 8 apart,
  // inside one 128 MB chunk plane instead of one 8.5 MB x plane per position.
  // (measured against [kz chunk][y][x][8], which makes P1's stores contiguous
  // instead: P1 22.2 -> 21.4 ms but P2 20.6 -> 21.8 ms)
  long long cm_xs() const { return static_cast<long long>(lo.spec_shape[1]) * 8; }
  long long cm_ys() const { return 8; }
  ColGeom cm_xout() const {  // P1 output: rows = y, positions = x
    ColGeom g = xgeom();
    g.rs = cm_ys();
    g.ps0 = cm_xs();
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[0]) * lo.spec_shape[1] * 8;
    g.mrows = static_cast<int>(lo.spec_shape[1]);
    return g;
  }
  ColGeom cm_y() const {  // y passes: rows = x, positions = y
    ColGeom g;
    g.rs = cm_xs();
    g.ps0 = cm_ys();
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[0]) * lo.spec_shape[1] * 8;
    g.nrows = static_cast<int>(lo.spec_shape[0]);
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = static_cast<int>(lo.spec_shape[0]);
    return g;
  }
  ColGeom cm_y_fwd() const {  // forward y pass, pruned like ygeom_fwd
    ColGeom g = cm_y();
    if (!cfg.dealias) return g;
    const int K = keep_k();
    const int kzk = std::max(0, std::min(g.n2, K + 1 - static_cast<int>(lo.spec_offset[2])));
    g.n2 = kzk;
    g.pitch = std::max(8, (kzk + 7) / 8 * 8);
    g.keep_k = K;
    return g;
  }
  ColGeom cm_x_fwd() const {  // forward x pass input: rows = y, positions = x
    ColGeom g = xgeom_fwd();   // (enumeration and pruning of the x layout)
    g.rs = cm_ys();
    g.ps0 = cm_xs();
    g.ps1 = 0;
    g.pb_shift = 30;
    g.kcs = static_cast<long long>(lo.spec_shape[0]) * lo.spec_shape[1] * 8;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = static_cast<int>(lo.spec_shape[1]);
    return g;
  }
  RowMap zmap_cm() const {  // z lines of the chunk-major layout: 128 B per kz chunk
    RowMap r = zmap(false);
    r.cstride = static_cast<int>(lo.spec_shape[0] * lo.spec_shape[1] * 8);
    r.xplane = static_cast<long long>(lo.spec_shape[1]) * 8;
    return r;
  }
  RowMap zmap_chunk() const {
    RowMap r = zmap(false);
    r.cstride = static_cast<int>(lo.spec_shape[1]) * 8;
    r.xplane = xpl();
    return r;
  }
  WaveGeom xwave() const {
    WaveGeom w;
    w.n = cfg.n;
    w.row_is_y = 1;
    w.row_off = static_cast<int>(lo.spec_offset[1]);
    w.kz_off = static_cast<int>(lo.spec_offset[2]);
    return w;
  }
  // y pass over the receive layout: rows = local x, positions = y
  ColGeom ygeom() const {
    ColGeom g;
    g.rs = plane();
    g.ps0 = pitch;
    g.ps1 = np * plane();
    g.pb_shift = ilog2(np);
    g.pblk = np;
    g.nrows = np;
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    g.mpitch = opt.ldgsts_tiles ? 0 : pitch;  // 0: no tensor map, LDGSTS tiles
    g.mrows = np;
    return g;
  }
  // Largest kept |k| of the 2/3 rule: |k| < n/3  <=>  |k| <= (n-1)/3
  // (dealias_mask, mesh.cpp:74-89).
  int keep_k() const { return (cfg.n - 1) / 3; }
  // Forward y pass: only kz < n/3 columns, only |ky| < n/3 outputs stored.
  ColGeom ygeom_fwd() const {
    ColGeom g = ygeom();
    if (!cfg.dealias) return g;
    const int K = keep_k();
    const int kzk = std::max(0, std::min(g.n2, K + 1 - static_cast<int>(lo.spec_offset[2])));
    g.n2 = kzk;
    g.pitch = std::max(8, (kzk + 7) / 8 * 8);
    g.keep_k = K;
    return g;
  }
  // Forward x pass: only (ky, kz) columns inside the 2/3 band, only |kx| < n/3
  // outputs stored. Local y rows form up to two kept bands.
  ColGeom xgeom_fwd() const {
    ColGeom g = xgeom();
    if (!cfg.dealias) return g;
    const int K = keep_k(), n = cfg.n;
    const int kzk = std::max(0, std::min(g.n2, K + 1 - static_cast<int>(lo.spec_offset[2])));
    g.n2 = kzk;
    g.pitch = std::max(8, (kzk + 7) / 8 * 8);
    g.keep_k = K;
    const int o1 = static_cast<int>(lo.spec_offset[1]), e1 = o1 + np;  // [o1, e1)
    const int a0 = std::max(o1, 0), a1 = std::min(e1, K + 1);             // [0, K]
    const int b0 = std::max(o1, n - K), b1 = std::min(e1, n);             // [n-K, n)
    const int na = std::max(0, a1 - a0), nb = std::max(0, b1 - b0);
    g.nrows = na + nb;
    g.seg_a = na;
    g.off0 = a0 - o1;
    g.off1 = b0 - o1;
    return g;
  }
  RowMap zmap(bool by_xy) const {
    RowMap r;
    r.n2 = static_cast<int>(lo.nf);
    if (pencil) {  // z lines (x_l, y_l) spread over the p2 kz segments of wd
      r.nrows = np * yl;
      r.nseg = static_cast<int>(seg_base.size());
      for (int q = 0; q < r.nseg; ++q) {
        r.seg_base[q] = seg_base[static_cast<size_t>(q)];
        r.seg_pitch[q] = seg_pitch[static_cast<size_t>(q)];
        r.seg_k0[q] = seg_k0[static_cast<size_t>(q)];
      }
      r.seg_k0[r.nseg] = r.n2;
      return r;
    }
    r.nrows = np * cfg.n;
    r.rpp = np;
    r.ny = cfg.n;
    r.blk = by_xy ? np : 0;
    r.prow = prow;
    r.pitch = pitch;
    return r;
  }
  // Pencil y pass over the row layout wc: element (x_l, y) at
  // ((y/yl)*np + x_l)*yl*pitch + (y%yl)*pitch.
  ColGeom ygeom_row() const {
    ColGeom g;
    g.rs = static_cast<long long>(yl) * pitch;
    g.ps0 = pitch;
    g.ps1 = static_cast<long long>(np) * yl * pitch;
    g.pb_shift = ilog2(yl);
    g.pblk = yl;
    g.nrows = np;
    g.n2 = static_cast<int>(lo.spec_shape[2]);
    g.pitch = pitch;
    return g;
  }
  // Peer-direct transposes over `grp` (slab: the world; pencil: the column
  // group, whose transposes move x blocks <-> y blocks exactly like the
  // slab's): map every member's wb and wa and build the store offsets
  // d_seg = [inverse (wb) | forward (wa)], member q's block for this rank
  // at its offset grp->rank() * blk. Collective over grp; the all_to_all
  // option or a transport that cannot map keeps the all-to-all.
  void map_peer_blocks(Comm* grp, int gp) {
    if (gp <= 1 || opt.all_to_all) return;
    peer_wb = grp->map_peers(wb);
    peer_wa = grp->map_peers(wa);
    if (peer_wb.empty() || peer_wa.empty()) {
      grp->unmap_peers(peer_wb);
      grp->unmap_peers(peer_wa);
      peer_wb.clear();
      peer_wa.clear();
      return;
    }
    const long long blk = static_cast<long long>(np) * plane();
    const long long me = grp->rank();
    std::vector<long long> seg(2 * static_cast<size_t>(gp));
    auto delta = [](void* a, void* b) {
      return static_cast<long long>((reinterpret_cast<intptr_t>(a) -
                                     reinterpret_cast<intptr_t>(b)) /
                                    static_cast<intptr_t>(sizeof(double2)));
    };
    for (int q = 0; q < gp; ++q) {
      seg[q] = delta(peer_wb[q], wb) + me * blk;
      seg[gp + q] = delta(peer_wa[q], wa) + me * blk;
    }
    SDNS_CUDA(cudaMalloc(&d_seg, sizeof(long long) * seg.size()));
    SDNS_CUDA(cudaMemcpyAsync(d_seg, seg.data(), sizeof(long long) * seg.size(),
                              cudaMemcpyHostToDevice, stream));
    peer_grp = grp;
    peer_n = gp;
    peer = true;
  }
  // Pencil row group (same coord1, ordered by coord2 = its kz block): map
  // the members' wd and wc; collective over the row group.
  void map_row_peers() {
    const int p2 = cfg.p2;
    if (!pencil || p2 <= 1 || opt.all_to_all) return;
    peer_wd = row->map_peers(wd);
    peer_wc = row->map_peers(wc);
    if (peer_wd.empty() || peer_wc.empty()) {
      row->unmap_peers(peer_wd);
      row->unmap_peers(peer_wc);
      peer_wd.clear();
      peer_wc.clear();
      return;
    }
    auto delta = [](void* a, void* b) {
      return static_cast<long long>((reinterpret_cast<intptr_t>(a) -
                                     reinterpret_cast<intptr_t>(b)) /
                                    static_cast<intptr_t>(sizeof(double2)));
    };
    const int me = row->rank();
    const long long rows = static_cast<long long>(np) * yl;
    std::vector<long long> seg(static_cast<size_t>(p2));
    RowMap r = zmap(false);
    for (int q = 0; q < p2; ++q) {
      const size_t uq = static_cast<size_t>(q);
      seg[uq] = delta(peer_wd[uq], wd) + seg_base[static_cast<size_t>(me)];
      r.seg_base[q] = delta(peer_wc[uq], wc) + me * rows * seg_pitch[uq];
      r.seg_pitch[q] = seg_pitch[uq];
      r.seg_cs[q] = rows * p2 * seg_pitch[uq];
    }
    zmo_row = r;
    SDNS_CUDA(cudaMalloc(&d_seg_row, sizeof(long long) * seg.size()));
    SDNS_CUDA(cudaMemcpyAsync(d_seg_row, seg.data(), sizeof(long long) * seg.size(),
                              cudaMemcpyHostToDevice, stream));
    peer_row = true;
  }
  // Pencil column-group transpose, wa <-> wb (x blocks <-> y2 blocks),
  // fft.cpp:166-173 / :191-199 without the pack/unpack passes.
  void exchange_col(bool inverse_dir, int nfields) {
    const int tk = tick(inverse_dir ? SDNS_PASS_A2A_INV : SDNS_PASS_A2A_FWD);
    const long long blk = np * plane();
    std::vector<Xfer> xs;
    double2* src = inverse_dir ? wa : wb;
    double2* dst = inverse_dir ? wb : wa;
    for (int f = 0; f < nfields; ++f)
      for (int s = 0; s < cfg.p1; ++s) {
        const long long off = f * spec_cs + s * blk;
        const size_t bytes = sizeof(double2) * static_cast<size_t>(blk);
        xs.push_back({s, src + off, dst + off, bytes, bytes});
      }
    col->alltoall(xs, stream);
    tock(tk);
  }
  // Pencil row-group transpose, wc <-> wd: my kz block of every row peer's
  // y slice <-> every peer's kz block of my y slice (unequal blocks when
  // p2 does not divide n/2+1), fft.cpp:141-160 / :203-223.
  void exchange_row(bool inverse_dir, int nfields) {
    const int tk = tick(inverse_dir ? SDNS_PASS_A2A_INV : SDNS_PASS_A2A_FWD);
    const long long rows = static_cast<long long>(np) * yl;
    std::vector<Xfer> xs;
    for (int f = 0; f < nfields; ++f)
      for (int q = 0; q < cfg.p2; ++q) {
        double2* c = wc + f * cs_c + q * rows * pitch;
        double2* d = wd + f * cs_d + seg_base[static_cast<size_t>(q)];
        const size_t cb = sizeof(double2) * static_cast<size_t>(rows * pitch);
        const size_t db = sizeof(double2) * static_cast<size_t>(rows * seg_pitch[static_cast<size_t>(q)]);
        if (inverse_dir) xs.push_back({q, c, d, cb, db});
        else xs.push_back({q, d, c, db, cb});
      }
    row->alltoall(xs, stream);
    tock(tk);
  }
  // ncomp host components (RankLayout block order, contiguous) <-> the
  // padded device layout: one contiguous DMA through the free work buffer
  // plus an HBM-speed repack kernel (the copy engines move contiguous blocks
  // markedly faster than the 2-D pitched copy). Only between pipeline runs.
  void copy_spec_all(double2* dev, double* host, int ncomp, bool to_device) const {
    const size_t bytes = sizeof(double2) * static_cast<size_t>(lo.spec_shape[0]) *
                         static_cast<size_t>(lo.spec_shape[1]) *
                         static_cast<size_t>(lo.spec_shape[2]) * static_cast<size_t>(ncomp);
    double2* stage = wa;  // >= 6 padded components
    if (to_device) {
      SDNS_CUDA(cudaMemcpyAsync(stage, host, bytes, cudaMemcpyHostToDevice, stream));
      sdns_dev::pw_repack(stage, dev, ncomp, sgeom(), false, stream);
    } else {
      sdns_dev::pw_repack(dev, stage, ncomp, sgeom(), true, stream);
      SDNS_CUDA(cudaMemcpyAsync(host, stage, bytes, cudaMemcpyDeviceToHost, stream));
    }
  }
  // transpose between wa (x layout) and wb (receive layout)
  // Transpose of the fields `fl` on stream `st` (the overlapped pipeline).
  void exchange_fields(bool inverse_dir, std::initializer_list<int> fl, cudaStream_t st) {
    const int nf = *std::max_element(fl.begin(), fl.end()) + 1;
    const auto plan = exchange_plan(cfg, lo, inverse_dir, nf);
    std::vector<Xfer> xs;
    double2* src = inverse_dir ? wa : wb;
    double2* dst = inverse_dir ? wb : wa;
    const long long per = static_cast<long long>(plan.size()) / nf;  // entries per field
    for (int f : fl)
      for (long long q = 0; q < per; ++q) {
        const auto& e = plan[static_cast<size_t>(f * per + q)];
        const size_t bytes = sizeof(double2) * static_cast<size_t>(e[3]);
        xs.push_back({static_cast<int>(e[0]), src + e[1], dst + e[2], bytes, bytes});
      }
    world->alltoall(xs, st);
  }
  void exchange(bool inverse_dir, int nfields) {
    if (cfg.p == 1) return;
    const int tk = tick(inverse_dir ? SDNS_PASS_A2A_INV : SDNS_PASS_A2A_FWD);
    const auto plan = exchange_plan(cfg, lo, inverse_dir, nfields);
    std::vector<Xfer> xs;
    xs.reserve(plan.size());
    double2* src = inverse_dir ? wa : wb;
    double2* dst = inverse_dir ? wb : wa;
    for (const auto& e : plan) {
      const size_t bytes = sizeof(double2) * static_cast<size_t>(e[3]);
      xs.push_back({static_cast<int>(e[0]), src + e[1], dst + e[2], bytes, bytes});
    }
    world->alltoall(xs, stream);
    tock(tk);
  }
};

struct sdns_field {
  sdns_ctx* ctx = nullptr;
  int kind = SDNS_SPECTRAL;
  int ncomp = 0;
  void* data = nullptr;
  bool owned = true;
  double2* spec() const { return static_cast<double2*>(data); }
  double* real() const { return static_cast<double*>(data); }
};

struct sdns_state {
  sdns_ctx* ctx = nullptr;
  sdns_field u;        // current state (the reference's u_hat / base)
  double2* nxt = nullptr;    // stage value
  double2* accum = nullptr;
  double2* carry = nullptr;
  double t = 0.0;
  int64_t step = 0;
};

namespace {

// Every entry point starts here; see sdns_ctx::peer_fresh.
void set_device(sdns_ctx* c) {
  SDNS_CUDA(cudaSetDevice(c->device));
  c->peer_fresh = false;
}

void require_spec(const sdns_field* f, int ncomp, const char* what) {
  if (!f || f->kind != SDNS_SPECTRAL || f->ncomp < ncomp)
    config_error(std::string(what) + ": expected a spectral field with " + std::to_string(ncomp) +
                 " components");
}
void require_real(const sdns_field* f, int ncomp, const char* what) {
  if (!f || f->kind != SDNS_REAL || f->ncomp < ncomp)
    config_error(std::string(what) + ": expected a real field with " + std::to_string(ncomp) +
                 " components");
}

void post_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(SDNS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// One fused RHS evaluation: P1 .. P5 (kernels.cu) with the transposes.
// Pencil forward y pass geometry: reads the row layout (wc), writes the
// column-send layout (wb); with the 2/3 rule on only kz < n/3 columns are
// transformed and only |ky| < n/3 outputs stored.
void pencil_yfwd_geoms(const sdns_ctx* c, bool prune, ColGeom& gi, ColGeom& go) {
  gi = c->ygeom_row();
  go = c->ygeom();
  if (!prune || !c->cfg.dealias) return;
  const int K = c->keep_k();
  const int kzk = std::max(0, std::min(gi.n2, K + 1 - static_cast<int>(c->lo.spec_offset[2])));
  gi.n2 = kzk;
  gi.pitch = std::max(8, (kzk + 7) / 8 * 8);
  go.keep_k = K;
}

// Slab p > 1 with the transposes overlapped: P1 runs per input component
// (component c writes fields {c} or {c, 2 + c}); each group's transpose goes
// out on the comm stream while the next component transforms, and P2 runs
// per group as its data arrives. On the forward side P4 and P5a run per
// field around the per-field transposes. Kernels and arithmetic are those of
// the serial path, so results are bitwise identical.
void rhs_slab_overlap(sdns_ctx* c, const double2* u_in, int mode, const XfArgs& args_in) {
  const int n = c->cfg.n;
  cudaStream_t s = c->stream, cs = c->cstream;
  cudaEvent_t* ev = c->xev;
  const long long sc = c->spec_cs;
  int tk = c->tick(SDNS_PASS_X_INV_CURL);
  for (int g = 0; g < 3; ++g) {
    sdns_dev::x_inverse_split(n, u_in, sc, c->wa, sc, c->xgeom(), nullptr, c->tw, s, g, 1);
    SDNS_CUDA(cudaEventRecord(ev[g], s));
    SDNS_CUDA(cudaStreamWaitEvent(cs, ev[g], 0));
    if (g == 0) c->exchange_fields(true, {0}, cs);
    else if (g == 1) c->exchange_fields(true, {1, 3}, cs);
    else c->exchange_fields(true, {2, 4}, cs);
    SDNS_CUDA(cudaEventRecord(ev[3 + g], cs));
  }
  c->tock(tk);
  tk = c->tick(SDNS_PASS_Y_INV);
  const int item_lo[3] = {0, 1, 3}, item_cnt[3] = {1, 2, 2};
  for (int g = 0; g < 3; ++g) {
    SDNS_CUDA(cudaStreamWaitEvent(s, ev[3 + g], 0));
    sdns_dev::y_inverse_curl(n, c->wb, sc, c->ygeom(), c->tw, s, item_lo[g], item_cnt[g]);
  }
  c->tock(tk);
  RowMap zm = c->zmap(false);
  if (c->cfg.dealias) zm.kz_keep = c->keep_k() + 1;
  tk = c->tick(SDNS_PASS_Z_FUSED);
  sdns_dev::z_fused(n, c->wb, sc, zm, c->norm, c->tw, s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_Y_FWD);
  for (int f = 0; f < 3; ++f) {
    sdns_dev::col_plain(n, -1, false, c->wb + f * sc, c->wb + f * sc, sc, sc, 1, c->ygeom_fwd(),
                        c->tw, s);
    SDNS_CUDA(cudaEventRecord(ev[6 + f], s));
    SDNS_CUDA(cudaStreamWaitEvent(cs, ev[6 + f], 0));
    c->exchange_fields(false, {f}, cs);
    SDNS_CUDA(cudaEventRecord(ev[9 + f], cs));
  }
  c->tock(tk);
  XfArgs a = args_in;
  a.nl = c->wa;
  a.nl_cs = sc;
  a.cs = sc;
  a.dealias = c->cfg.dealias;
  tk = c->tick(SDNS_PASS_X_FWD_FFT);
  for (int f = 0; f < 3; ++f) {
    SDNS_CUDA(cudaStreamWaitEvent(s, ev[9 + f], 0));
    sdns_dev::col_plain(n, -1, true, c->wa + f * sc, c->wa + f * sc, sc, sc, 1, c->xgeom_fwd(),
                        c->tw, s);
  }
  c->tock(tk);
  tk = c->tick(SDNS_PASS_X_FWD_TAIL + mode);
  sdns_dev::rk_update(mode, a, c->sgeom(), s);
  c->tock(tk);
  post_launch("rhs pipeline (overlapped transposes)");
}

// Slab p > 1 with peer-direct transposes: the transposes are fused into the
// passes that produce their data. P1 stores each output x plane straight into
// the receive layout of the rank that owns it (same device, or NVLink through
// a CUDA IPC mapping), and P4 stores each y output into the owner's x
// layout, so no all-to-all pass, staging buffer or copy engine is involved;
// a stream barrier across the ranks follows each (its wait also orders the
// next write into a buffer after the owner's last read of it: wb is last read
// by P4 before the forward barrier, wa by P5 before the next inverse one).
// The transforms are the serial path's, so results are bitwise identical.
void rhs_slab_peer(sdns_ctx* c, const double2* u_in, int mode, const XfArgs& args_in) {
  const int n = c->cfg.n, p = c->peer_n;
  cudaStream_t s = c->stream;
  const long long sc = c->spec_cs;
  int tk = c->tick(SDNS_PASS_X_INV_CURL);
  ColGeom go1 = c->xgeom();
  go1.pb_shift = ilog2(c->np);
  go1.pblk = c->np;
  go1.ps1 = 0;
  go1.seg = c->d_seg;
  sdns_dev::x_inverse_split(n, u_in, sc, c->wb, sc, c->xgeom(), &go1, c->tw, s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_A2A_INV);
  c->peer_grp->stream_barrier(s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_Y_INV);
  sdns_dev::y_inverse_curl(n, c->wb, sc, c->ygeom(), c->tw, s);
  c->tock(tk);
  RowMap zm = c->zmap(false);
  if (c->cfg.dealias) zm.kz_keep = c->keep_k() + 1;
  tk = c->tick(SDNS_PASS_Z_FUSED);
  sdns_dev::z_fused(n, c->wb, sc, zm, c->norm, c->tw, s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_Y_FWD);
  const ColGeom gi4 = c->ygeom_fwd();
  ColGeom go4 = gi4;
  go4.ps1 = 0;
  go4.seg = c->d_seg + p;
  sdns_dev::col_plain_to(n, -1, c->wb, c->wa, sc, sc, 3, gi4, go4, c->tw, s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_A2A_FWD);
  c->peer_grp->stream_barrier(s);
  c->tock(tk);
  XfArgs a = args_in;
  a.nl = c->wa;
  a.nl_cs = sc;
  a.cs = sc;
  a.dealias = c->cfg.dealias;
  tk = c->tick(SDNS_PASS_X_FWD_FFT);
  sdns_dev::col_plain(n, -1, true, c->wa, c->wa, sc, sc, 3, c->xgeom_fwd(), c->tw, s);
  c->tock(tk);
  tk = c->tick(SDNS_PASS_X_FWD_TAIL + mode);
  sdns_dev::rk_update(mode, a, c->sgeom(), s);
  c->tock(tk);
  post_launch("rhs pipeline (peer-direct transposes)");
}

// One fused RHS evaluation: P1 .. P5 (kernels*.cu) with the transposes.
void rhs_pipeline(sdns_ctx* c, const double2* u_in, int mode, const XfArgs& args_in) {
  if ((c->peer || c->peer_row) && !c->peer_fresh) {
    const int tb = c->tick(SDNS_PASS_A2A_INV);
    c->world->stream_barrier(c->stream);
    c->tock(tb);
  }
  c->peer_fresh = c->peer || c->peer_row;
  if (c->peer && !c->pencil) {
    rhs_slab_peer(c, u_in, mode, args_in);
    return;
  }
  if (c->cstream) {
    rhs_slab_overlap(c, u_in, mode, args_in);
    return;
  }
  const int n = c->cfg.n;
  cudaStream_t s = c->stream;
  int tk = c->tick(SDNS_PASS_X_INV_CURL);
  if (c->wx) {
    const ColGeom go = c->xl_out();
    sdns_dev::x_inverse_split(n, u_in, c->spec_cs, c->wx, c->cs_x, c->xgeom(), &go, c->tw, s);
  } else if (c->cmx) {
    const ColGeom go = c->cm_xout();
    sdns_dev::x_inverse_split(n, u_in, c->spec_cs, c->wa, c->spec_cs, c->xgeom(), &go, c->tw, s);
  } else if (c->peer) {  // pencil: P1 stores into the column peers' wb (see rhs_slab_peer)
    ColGeom go1 = c->xgeom();
    go1.pb_shift = ilog2(c->np);
    go1.pblk = c->np;
    go1.ps1 = 0;
    go1.seg = c->d_seg;
    sdns_dev::x_inverse_split(n, u_in, c->spec_cs, c->wb, c->spec_cs, c->xgeom(), &go1, c->tw, s);
  } else {
    sdns_dev::x_inverse_split(n, u_in, c->spec_cs, c->wa, c->spec_cs, c->xgeom(), nullptr, c->tw,
                              s);
  }
  c->tock(tk);
  // Forward direction: with the 2/3 rule on, modes the mask zeroes are never
  // computed or stored (kept modes are computed by identical transforms).
  RowMap zm = c->zmap(false);
  if (c->cfg.dealias) zm.kz_keep = c->keep_k() + 1;
  if (!c->pencil) {
    if (c->wx) {
      tk = c->tick(SDNS_PASS_Y_INV);
      sdns_dev::y_inverse_curl_to(n, c->wx, c->wb, c->cs_x, c->spec_cs, c->xl_in(),
                                  c->zchunk ? c->yc_geom() : c->ygeom(), c->tw, s);
    } else if (c->cmx) {
      tk = c->tick(SDNS_PASS_Y_INV);
      sdns_dev::y_inverse_curl(n, c->wa, c->spec_cs, c->cm_y(), c->tw, s);
    } else {
      c->exchange(true, 5);
      tk = c->tick(SDNS_PASS_Y_INV);
      sdns_dev::y_inverse_curl(n, c->wb, c->spec_cs, c->ygeom(), c->tw, s);
    }
    c->tock(tk);
    tk = c->tick(SDNS_PASS_Z_FUSED);
    if (c->cmx) {
      RowMap zc = c->zmap_cm();
      zc.kz_keep = zm.kz_keep;
      sdns_dev::z_fused(n, c->wa, c->spec_cs, zc, c->norm, c->tw, s);
    } else if (c->zchunk) {
      RowMap zc = c->zmap_chunk();
      zc.kz_keep = zm.kz_keep;
      sdns_dev::z_fused(n, c->wb, c->spec_cs, zc, c->norm, c->tw, s);
    } else {
      sdns_dev::z_fused(n, c->wb, c->spec_cs, zm, c->norm, c->tw, s);
    }
    c->tock(tk);
    tk = c->tick(SDNS_PASS_Y_FWD);
    sdns_dev::col_plain(n, -1, false, c->wb, c->wb, c->spec_cs, c->spec_cs, 3,
                        c->cmx ? c->cm_y_fwd() : (c->zchunk ? c->yc_geom_fwd() : c->ygeom_fwd()),
                        c->tw, s);
    c->tock(tk);
    c->exchange(false, 3);
  } else {
    if (c->peer) {
      const int tb = c->tick(SDNS_PASS_A2A_INV);
      c->peer_grp->stream_barrier(s);
      c->tock(tb);
    } else {
      c->exchange_col(true, 5);
    }
    if (c->peer_row) {  // the row transposes fused into P2 and the z pass
      ColGeom go2 = c->ygeom_row();
      go2.ps1 = 0;
      go2.seg = c->d_seg_row;
      tk = c->tick(SDNS_PASS_Y_INV);
      sdns_dev::y_inverse_curl_to(n, c->wb, c->wd, c->spec_cs, c->cs_d, c->ygeom(), go2, c->tw,
                                  s);
      c->tock(tk);
      int tb = c->tick(SDNS_PASS_A2A_INV);
      c->row->stream_barrier(s);
      c->tock(tb);
      tk = c->tick(SDNS_PASS_Z_FUSED);
      RowMap zo = c->zmo_row;
      zo.kz_keep = zm.kz_keep;
      sdns_dev::z_fused_to(n, c->wd, c->cs_d, zm, c->wc, zo, c->norm, c->tw, s);
      c->tock(tk);
      tb = c->tick(SDNS_PASS_A2A_FWD);
      c->row->stream_barrier(s);
      c->tock(tb);
    } else {
      tk = c->tick(SDNS_PASS_Y_INV);
      sdns_dev::y_inverse_curl_to(n, c->wb, c->wc, c->spec_cs, c->cs_c, c->ygeom(),
                                  c->ygeom_row(), c->tw, s);
      c->tock(tk);
      c->exchange_row(true, 6);
      tk = c->tick(SDNS_PASS_Z_FUSED);
      sdns_dev::z_fused(n, c->wd, c->cs_d, zm, c->norm, c->tw, s);
      c->tock(tk);
      c->exchange_row(false, 3);
    }
    ColGeom gi, go;
    pencil_yfwd_geoms(c, true, gi, go);
    tk = c->tick(SDNS_PASS_Y_FWD);
    if (c->peer) {  // P4 stores into the column peers' x layouts (wa)
      go.ps1 = 0;
      go.seg = c->d_seg + c->peer_n;
      sdns_dev::col_plain_to(n, -1, c->wc, c->wa, c->cs_c, c->spec_cs, 3, gi, go, c->tw, s);
      c->tock(tk);
      const int tb = c->tick(SDNS_PASS_A2A_FWD);
      c->peer_grp->stream_barrier(s);
      c->tock(tb);
    } else {
      sdns_dev::col_plain_to(n, -1, c->wc, c->wb, c->cs_c, c->spec_cs, 3, gi, go, c->tw, s);
      c->tock(tk);
      c->exchange_col(false, 3);
    }
  }
  XfArgs a = args_in;
  a.nl = c->wa;
  a.nl_cs = c->spec_cs;
  a.cs = c->spec_cs;
  a.dealias = c->cfg.dealias;
  tk = c->tick(SDNS_PASS_X_FWD_FFT);
  if (c->zchunk || c->cmx) {  // chunked input, x-layout output in the free fields 3..5
    a.nl = c->wa + 3 * c->spec_cs;
    sdns_dev::col_plain_to(n, -1, c->wa, c->wa + 3 * c->spec_cs, c->spec_cs, c->spec_cs, 3,
                           c->cmx ? c->cm_x_fwd() : c->xc_geom_fwd(), c->xgeom_fwd(), c->tw, s,
                           true);
  } else {
    sdns_dev::col_plain(n, -1, true, c->wa, c->wa, c->spec_cs, c->spec_cs, 3, c->xgeom_fwd(),
                        c->tw, s);
  }
  c->tock(tk);
  tk = c->tick(SDNS_PASS_X_FWD_TAIL + mode);
  sdns_dev::rk_update(mode, a, c->sgeom(), s);
  c->tock(tk);
  post_launch("rhs pipeline");
}

void fft_forward_impl(sdns_ctx* c, const sdns_field* real, sdns_field* spec) {
  const int n = c->cfg.n;
  cudaStream_t s = c->stream;
  const int nc = std::min(real->ncomp, spec->ncomp);
  if (!c->pencil) {
    for (int f = 0; f < nc; ++f)
      sdns_dev::z_r2c(n, real->real() + f * c->real_cs, c->wb + f * c->spec_cs, c->zmap(true),
                      c->tw, s);
    if (c->peer) {  // the y pass stores into the owners' x layouts
      c->world->stream_barrier(s);  // the peers are done with their wa
      ColGeom go = c->ygeom();
      go.ps1 = 0;
      go.seg = c->d_seg + c->peer_n;
      sdns_dev::col_plain_to(n, -1, c->wb, c->wa, c->spec_cs, c->spec_cs, nc, c->ygeom(), go,
                             c->tw, s);
      c->world->stream_barrier(s);
    } else {
      sdns_dev::col_plain(n, -1, false, c->wb, c->wb, c->spec_cs, c->spec_cs, nc, c->ygeom(),
                          c->tw, s);
      c->exchange(false, nc);
    }
  } else {
    if (c->peer_row) {  // z r2c stores each kz segment into its owner's wc
      c->row->stream_barrier(s);  // the row peers are done with their wc
      for (int f = 0; f < nc; ++f)
        sdns_dev::z_r2c_to(n, real->real() + f * c->real_cs, c->wc, c->zmap(true), c->zmo_row, f,
                           c->tw, s);
      c->row->stream_barrier(s);
    } else {
      for (int f = 0; f < nc; ++f)
        sdns_dev::z_r2c(n, real->real() + f * c->real_cs, c->wd + f * c->cs_d, c->zmap(true),
                        c->tw, s);
      c->exchange_row(false, nc);
    }
    ColGeom gi, go;
    pencil_yfwd_geoms(c, false, gi, go);
    if (c->peer) {  // the y pass stores into the column owners' x layouts
      c->col->stream_barrier(s);
      go.ps1 = 0;
      go.seg = c->d_seg + c->peer_n;
      sdns_dev::col_plain_to(n, -1, c->wc, c->wa, c->cs_c, c->spec_cs, nc, gi, go, c->tw, s);
      c->col->stream_barrier(s);
    } else {
      sdns_dev::col_plain_to(n, -1, c->wc, c->wb, c->cs_c, c->spec_cs, nc, gi, go, c->tw, s);
      c->exchange_col(false, nc);
    }
  }
  sdns_dev::col_plain(n, -1, true, c->wa, spec->spec(), c->spec_cs, c->spec_cs, nc, c->xgeom(),
                      c->tw, s);
  post_launch("fft forward");
}

void fft_inverse_impl(sdns_ctx* c, const sdns_field* spec, sdns_field* real) {
  const int n = c->cfg.n;
  cudaStream_t s = c->stream;
  const int nc = std::min(real->ncomp, spec->ncomp);
  if (c->peer) {  // the x pass stores into the (column) owners' receive layouts
    c->peer_grp->stream_barrier(s);  // the peers are done with their wb
    ColGeom go = c->xgeom();
    go.pb_shift = ilog2(c->np);
    go.pblk = c->np;
    go.ps1 = 0;
    go.seg = c->d_seg;
    sdns_dev::col_plain_to(n, +1, spec->spec(), c->wb, c->spec_cs, c->spec_cs, nc, c->xgeom(), go,
                           c->tw, s, true);
    c->peer_grp->stream_barrier(s);
  } else {
    sdns_dev::col_plain(n, +1, true, spec->spec(), c->wa, c->spec_cs, c->spec_cs, nc, c->xgeom(),
                        c->tw, s);
  }
  if (!c->pencil) {
    if (!c->peer) c->exchange(true, nc);
    sdns_dev::col_plain(n, +1, false, c->wb, c->wb, c->spec_cs, c->spec_cs, nc, c->ygeom(), c->tw,
                        s);
    for (int f = 0; f < nc; ++f)
      sdns_dev::z_c2r(n, c->wb + f * c->spec_cs, real->real() + f * c->real_cs, c->zmap(true),
                      c->norm, c->tw, s);
  } else {
    if (!c->peer) c->exchange_col(true, nc);
    if (c->peer_row) {  // the y pass stores its y blocks into the row owners' z lines
      c->row->stream_barrier(s);  // the row peers are done with their wd
      ColGeom go = c->ygeom_row();
      go.ps1 = 0;
      go.seg = c->d_seg_row;
      sdns_dev::col_plain_to(n, +1, c->wb, c->wd, c->spec_cs, c->cs_d, nc, c->ygeom(), go, c->tw,
                             s);
      c->row->stream_barrier(s);
    } else {
      sdns_dev::col_plain_to(n, +1, c->wb, c->wc, c->spec_cs, c->cs_c, nc, c->ygeom(),
                             c->ygeom_row(), c->tw, s);
      c->exchange_row(true, nc);
    }
    for (int f = 0; f < nc; ++f)
      sdns_dev::z_c2r(n, c->wd + f * c->cs_d, real->real() + f * c->real_cs, c->zmap(true),
                      c->norm, c->tw, s);
  }
  post_launch("fft inverse");
}

// The four stages of one step (device work only; see step_impl).
void step_stages(sdns_ctx* c, sdns_state* st, double dt, int post_project, bool want_stats,
                 const double* dts = nullptr) {
  static const double kW[3] = {1.0, 2.0, 2.0};
  static const double kB[3] = {0.5, 0.5, 1.0};
  double2* u = st->u.spec();
  for (int stage = 0; stage < 4; ++stage) {
    XfArgs a{};
    a.nu = c->cfg.nu;
    a.base = u;
    a.cs = c->spec_cs;
    a.dts = dts;
    a.dts_stage = stage;
    if (stage < 3) {
      a.u = stage == 0 ? u : st->nxt;
      a.out = st->nxt;
      a.accum = st->accum;
      a.w = kW[stage];
      a.bdt = kB[stage] * dt;
      // stage 1: u_1 = u0 + b0 dt du_0 and accum = 1 * du_0 hold the same bits
      // the stage-0 update wrote, so the update rebuilds u_1 instead of reading it
      if (stage == 1) a.ubdt = kB[0] * dt;
      rhs_pipeline(c, a.u, stage == 0 ? sdns_dev::XF_RK0 : sdns_dev::XF_RK12, a);
    } else {
      a.u = st->nxt;
      a.accum = st->accum;
      a.carry = st->carry;
      a.base_out = u;
      a.sixth = dt / 6.0;
      a.project = post_project;
      a.finite = c->d_flag;
      if (want_stats) {
        a.stats_partial = c->d_fpartial;
        a.stats_out = c->d_fout;
        a.shells = c->shells;
      }
      SDNS_CUDA(cudaMemsetAsync(c->d_flag, 0xff, sizeof(int), c->stream));
      rhs_pipeline(c, st->nxt, sdns_dev::XF_RK3, a);
    }
  }
}

// One RK4 step. On a single rank (no collectives inside the step) the
// stages replay as a CUDA graph captured once per (state, dt, flags): the
// ~25 launches of a step cost one graph launch, which matters where the
// kernels are short (64^3: config 1). Per-pass timing runs eagerly.
bool step_impl(sdns_ctx* c, sdns_state* st, double dt, int post_project, bool want_flag,
               bool want_stats = false) {
  const bool graph = c->cfg.p == 1 && !c->timing && !c->opt.no_graph;
  if (!graph) {
    step_stages(c, st, dt, post_project, want_stats);
  } else {
    sdns_ctx::StepGraph& g = c->graphs[want_stats ? 1 : 0];
    // dt is a device-side scalar of the captured step (advance's dt_k varies
    // in its last bits from step to step)
    sdns_dev::set_step_scalars(c->d_dts, dt, c->stream);
    if (!g.exec || g.st != st || g.post_project != post_project) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
      cudaGraph_t graph_def = nullptr;
      SDNS_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        step_stages(c, st, dt, post_project, want_stats, c->d_dts);
      } catch (...) {
        cudaStreamEndCapture(c->stream, &graph_def);
        if (graph_def) cudaGraphDestroy(graph_def);
        throw;
      }
      SDNS_CUDA(cudaStreamEndCapture(c->stream, &graph_def));
      SDNS_CUDA(cudaGraphInstantiate(&g.exec, graph_def, 0));
      cudaGraphDestroy(graph_def);
      g.st = st;
      g.post_project = post_project;
    }
    SDNS_CUDA(cudaGraphLaunch(g.exec, c->stream));
  }
  st->t += dt;
  st->step += 1;
  c->fused_on_host = false;
  if (!want_flag) return true;
  SDNS_CUDA(cudaMemcpyAsync(c->h_flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (want_stats)
    SDNS_CUDA(cudaMemcpyAsync(c->h_fout, c->d_fout, sizeof(double) * (c->shells + 3),
                              cudaMemcpyDeviceToHost, c->stream));
  c->wait();
  c->fused_on_host = want_stats;
  double ok = *c->h_flag != 0 ? 1.0 : 0.0;
  c->world->allreduce(&ok, 1, 2);
  return ok > 0.5;
}

void stats_impl(sdns_ctx* c, const sdns_field* u, double nu, double t, double* row) {
  const SpecGeom g = c->sgeom();
  const double* src = c->d_fout;
  const double* h = c->h_out;
  if (u == c->fused_u && c->fused_on_host) {
    h = c->h_fout;  // fetched with the step's finite flag
  } else {
    if (u != c->fused_u) {
      sdns_dev::stats_local(u->spec(), g, c->shells, c->d_partial, c->d_out, c->stream);
      post_launch("collect_stats");
      src = c->d_out;
    }
    const int stride = c->shells + 3;
    SDNS_CUDA(cudaMemcpyAsync(c->h_out, src, sizeof(double) * stride, cudaMemcpyDeviceToHost,
                              c->stream));
    c->wait();
  }
  std::vector<double> sums(static_cast<size_t>(2 + c->shells));
  sums[0] = h[0];
  sums[1] = h[1];
  for (int i = 0; i < c->shells; ++i) sums[2 + i] = h[3 + i];
  double dmax = h[2];
  c->world->allreduce(sums.data(), static_cast<int>(sums.size()), 0);
  c->world->allreduce(&dmax, 1, 1);
  const double n3 = static_cast<double>(c->cfg.n) * c->cfg.n * c->cfg.n;
  const double n6 = n3 * n3;
  row[0] = t;
  row[1] = 0.5 * sums[0] / n6;
  row[2] = 0.5 * sums[1] / n6;
  row[3] = 2.0 * nu * row[2];
  row[4] = dmax;
  for (int i = 0; i < c->shells; ++i) row[5 + i] = sums[2 + i] / n6;
}

// ---- checkpoints (checkpoint.cpp:64-187) --------------------------------

constexpr char kCkMagic[4] = {'S', 'D', 'N', 'S'};
constexpr uint32_t kCkVersion = 1;
struct CkHeader {
  char magic[4];
  uint32_t version;
  uint32_t n;
  uint32_t components;
  double t;
  uint64_t step;
};
static_assert(sizeof(CkHeader) == 32, "reference checkpoint header is 32 bytes");

// Root's verdict to every rank, as the reference shares it (length, then
// the bytes, by broadcast_bytes; checkpoint.cpp:104-110): a bad path or file
// raises IoError on every rank instead of hanging the others.
void share_io_error(sdns_ctx* c, const std::string& root_err) {
  uint64_t len = c->world->rank() == 0 ? root_err.size() : 0;
  c->world->broadcast(&len, sizeof(len), 0);
  if (len == 0) return;
  std::string m = c->world->rank() == 0 ? root_err : std::string(static_cast<size_t>(len), ' ');
  c->world->broadcast(m.data(), static_cast<size_t>(len), 0);
  throw Error(SDNS_IO_ERROR, m);
}

// Copies one rank's row-major real block into / out of the global x-major
// array (blit_block, checkpoint.cpp:45-60).
void blit_block(const sdns_layout& rl, int64_t n, double* global, double* block, bool to_global) {
  const int64_t s0 = rl.real_shape[0], s1 = rl.real_shape[1], s2 = rl.real_shape[2];
  for (int64_t i = 0; i < s0; ++i)
    for (int64_t j = 0; j < s1; ++j) {
      double* g = global + ((rl.real_offset[0] + i) * n + (rl.real_offset[1] + j)) * n +
                  rl.real_offset[2];
      double* b = block + (i * s1 + j) * s2;
      if (to_global) std::memcpy(g, b, sizeof(double) * static_cast<size_t>(s2));
      else std::memcpy(b, g, sizeof(double) * static_cast<size_t>(s2));
    }
}

// Gather (to_root) or scatter of one real component between every rank's
// block and rank 0's device staging buffer `stage` (blocks in rank order).
void ck_exchange(sdns_ctx* c, const std::vector<int64_t>& cnt, double* mine, double* stage,
                 bool to_root) {
  const int p = c->cfg.p;
  const bool root = c->world->rank() == 0;
  const size_t my = sizeof(double) * static_cast<size_t>(c->real_cs);
  std::vector<Xfer> xs;
  int64_t off = 0;
  for (int q = 0; q < p; ++q) {
    const size_t qb = sizeof(double) * static_cast<size_t>(cnt[static_cast<size_t>(q)]);
    double* slot = root ? stage + off : nullptr;
    if (to_root)
      xs.push_back({q, q == 0 ? mine : nullptr, slot, q == 0 ? my : 0, root ? qb : 0});
    else
      xs.push_back({q, slot, q == 0 ? mine : nullptr, root ? qb : 0, q == 0 ? my : 0});
    off += cnt[static_cast<size_t>(q)];
  }
  c->world->alltoall(xs, c->stream);
  c->wait();
}

// Root-side resources of a checkpoint transfer, released on every exit path.
struct CkRoot {
  FILE* fp = nullptr;
  double* stage = nullptr;  // device: one gathered component (n^3 doubles)
  ~CkRoot() {
    if (fp) std::fclose(fp);
    if (stage) cudaFree(stage);
  }
};

std::vector<int64_t> ck_counts(const sdns_ctx* c, std::vector<sdns_layout>& lays) {
  std::vector<int64_t> cnt;
  for (int r = 0; r < c->cfg.p; ++r) {
    lays.push_back(build_layout(c->cfg, r));
    cnt.push_back(lays.back().real_shape[0] * lays.back().real_shape[1] * lays.back().real_shape[2]);
  }
  return cnt;
}

// write_checkpoint (checkpoint.cpp:64-113): the root opens the file, writes
// the header and allocates its staging buffers BEFORE any collective, then
// shares the verdict; components are gathered to the root and written in
// global x-major order.
void checkpoint_write_impl(sdns_ctx* c, const sdns_field* u, const std::string& path, double t,
                           int64_t step) {
  const int64_t n = c->cfg.n, n3 = n * n * n;
  const bool root = c->world->rank() == 0;
  std::vector<sdns_layout> lays;
  const std::vector<int64_t> cnt = ck_counts(c, lays);
  CkRoot rs;
  std::vector<double> blocks, global;
  std::string err;
  if (root) {
    try {
      try {
        const auto dir = std::filesystem::path(path).parent_path();
        if (!dir.empty()) std::filesystem::create_directories(dir);
      } catch (const std::exception&) {
      }
      rs.fp = std::fopen(path.c_str(), "wb");
      if (!rs.fp) throw Error(SDNS_IO_ERROR, "cannot open checkpoint '" + path + "' for writing");
      CkHeader h{};
      std::memcpy(h.magic, kCkMagic, 4);
      h.version = kCkVersion;
      h.n = static_cast<uint32_t>(n);
      h.components = 3;
      h.t = t;
      h.step = static_cast<uint64_t>(step);
      if (std::fwrite(&h, sizeof(h), 1, rs.fp) != 1)
        throw Error(SDNS_IO_ERROR, "short write to checkpoint '" + path + "'");
      if (cudaMalloc(&rs.stage, sizeof(double) * static_cast<size_t>(n3)) != cudaSuccess) {
        cudaGetLastError();
        rs.stage = nullptr;
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': cannot allocate the " +
                                       std::to_string(8 * n3) + "-byte device staging buffer");
      }
      blocks.resize(static_cast<size_t>(n3));
      global.resize(static_cast<size_t>(n3));
    } catch (const std::exception& e) {
      err = e.what();
    }
  }
  share_io_error(c, err);
  bool ok = true;
  for (int comp = 0; comp < 3; ++comp) {
    ck_exchange(c, cnt, u->real() + comp * c->real_cs, rs.stage, true);
    if (!root) continue;
    SDNS_CUDA(cudaMemcpyAsync(blocks.data(), rs.stage, sizeof(double) * static_cast<size_t>(n3),
                              cudaMemcpyDeviceToHost, c->stream));
    c->wait();
    int64_t off = 0;
    for (int r = 0; r < c->cfg.p; ++r) {
      blit_block(lays[static_cast<size_t>(r)], n, global.data(), blocks.data() + off, true);
      off += cnt[static_cast<size_t>(r)];
    }
    ok = ok && std::fwrite(global.data(), sizeof(double), global.size(), rs.fp) == global.size();
  }
  if (root) {
    ok = (std::fclose(rs.fp) == 0) && ok;
    rs.fp = nullptr;
    if (!ok) throw Error(SDNS_IO_ERROR, "short write to checkpoint '" + path + "'");
  }
}

// read_checkpoint (checkpoint.cpp:115-187): the root validates and reads the
// whole file and allocates its staging buffer before any collective, shares
// the verdict, scatters every component (the host copy into the staging
// buffer is ordered on the context stream with the exchange), then t and
// step reach every rank by broadcast.
void checkpoint_read_impl(sdns_ctx* c, const std::string& path, sdns_field* u, double* t,
                          int64_t* step) {
  const int64_t n = c->cfg.n, n3 = n * n * n;
  const bool root = c->world->rank() == 0;
  std::vector<sdns_layout> lays;
  const std::vector<int64_t> cnt = ck_counts(c, lays);
  std::vector<double> global, blocks;
  CkHeader h{};
  CkRoot rs;
  std::string err;
  if (root) {
    try {
      rs.fp = std::fopen(path.c_str(), "rb");
      if (!rs.fp) throw Error(SDNS_IO_ERROR, "cannot open checkpoint '" + path + "'");
      if (std::fread(&h, sizeof(h), 1, rs.fp) != 1 || std::memcmp(h.magic, kCkMagic, 4) != 0)
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': bad magic");
      if (h.version != kCkVersion)
        throw Error(SDNS_IO_ERROR,
                    "checkpoint '" + path + "': unsupported version " + std::to_string(h.version));
      if (h.n != static_cast<uint32_t>(n))
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': grid size " + std::to_string(h.n) +
                                       " does not match configured n=" + std::to_string(n));
      if (h.components != 3)
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': expected 3 components");
      global.resize(static_cast<size_t>(3 * n3));
      if (std::fread(global.data(), sizeof(double), global.size(), rs.fp) != global.size())
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': truncated payload");
      std::fclose(rs.fp);
      rs.fp = nullptr;
      if (cudaMalloc(&rs.stage, sizeof(double) * static_cast<size_t>(n3)) != cudaSuccess) {
        cudaGetLastError();
        rs.stage = nullptr;
        throw Error(SDNS_IO_ERROR, "checkpoint '" + path + "': cannot allocate the " +
                                       std::to_string(8 * n3) + "-byte device staging buffer");
      }
      blocks.resize(static_cast<size_t>(n3));
    } catch (const std::exception& e) {
      err = e.what();
    }
  }
  share_io_error(c, err);
  for (int comp = 0; comp < 3; ++comp) {
    if (root) {
      int64_t off = 0;
      for (int r = 0; r < c->cfg.p; ++r) {
        blit_block(lays[static_cast<size_t>(r)], n, global.data() + comp * n3, blocks.data() + off,
                   false);
        off += cnt[static_cast<size_t>(r)];
      }
      SDNS_CUDA(cudaMemcpyAsync(rs.stage, blocks.data(), sizeof(double) * static_cast<size_t>(n3),
                                cudaMemcpyHostToDevice, c->stream));
    }
    ck_exchange(c, cnt, u->real() + comp * c->real_cs, rs.stage, false);
  }
  // every rank learns t and step from the root's header
  double meta[2] = {root ? h.t : 0.0, root ? static_cast<double>(h.step) : 0.0};
  c->world->broadcast(meta, sizeof(meta), 0);
  if (t) *t = meta[0];
  if (step) *step = static_cast<int64_t>(meta[1]);
}

void* dev_alloc(sdns_ctx* c, size_t bytes) {
  void* p = nullptr;
  SDNS_CUDA(cudaMalloc(&p, bytes));
  SDNS_CUDA(cudaMemsetAsync(p, 0, bytes, c->stream));
  c->dev_bytes += static_cast<int64_t>(bytes);
  return p;
}

}  // namespace

namespace sdns_host {
int run_guarded(const std::function<void()>& f) { return guarded(f); }
}  // namespace sdns_host

extern "C" {

const char* sdns_last_error(void) { return g_last_error.c_str(); }

const char* sdns_version(void) { return "sdns-b200 0.1 (sm_100a)"; }

int sdns_config_validate(const sdns_config* cfg) {
  return guarded([&] { validate(*cfg); });
}

int sdns_build_layout(const sdns_config* cfg, int rank, sdns_layout* out) {
  return guarded([&] { *out = build_layout(*cfg, rank); });
}

int sdns_device_layout(const sdns_config* cfg, int rank, sdns_dev_layout* out) {
  return guarded([&] { *out = dev_layout(*cfg, build_layout(*cfg, rank)); });
}

int sdns_exchange_plan(const sdns_config* cfg, int rank, int inverse, int nfields, int64_t* out,
                       int* count) {
  return guarded([&] {
    const auto plan = exchange_plan(*cfg, build_layout(*cfg, rank), inverse != 0, nfields);
    if (out)
      for (size_t i = 0; i < plan.size(); ++i)
        for (int j = 0; j < 4; ++j) out[4 * i + j] = plan[i][j];
    if (count) *count = static_cast<int>(plan.size());
  });
}

int64_t sdns_block_size(int64_t total, int parts, int index) { return block_size(total, parts, index); }
int64_t sdns_block_start(int64_t total, int parts, int index) { return block_start(total, parts, index); }
int64_t sdns_step_count(double t_end, double dt) { return step_count(t_end, dt); }
int sdns_spectrum_shells(int64_t n) { return spectrum_shells(n); }

int sdns_iso_init_host(int64_t n, uint64_t seed, double k0, double energy, const sdns_layout* lo,
                       double* out) {
  return guarded([&] {
    if (n < 4 || n % 2) config_error("iso init: n must be even and >= 4");
    iso_init(n, seed, k0, energy, *lo, out);
  });
}

int sdns_comm_loopback(sdns_comm** out) {
  return guarded([&] { *out = new sdns_comm{make_loopback_comm()}; });
}

int sdns_comm_inprocess_group(int size, int device, double timeout_s, sdns_comm** out) {
  return guarded([&] {
    auto g = make_inprocess_group(size, device, timeout_s);
    for (int r = 0; r < size; ++r) out[r] = new sdns_comm{g[static_cast<size_t>(r)]};
  });
}

int sdns_comm_nccl_unique_id(unsigned char id[128]) {
  return guarded([&] { nccl_unique_id(id); });
}

int sdns_comm_nccl_init(const unsigned char id[128], int size, int rank, int device, sdns_comm** out) {
  return guarded([&] { *out = new sdns_comm{make_nccl_comm(id, size, rank, device)}; });
}

int sdns_comm_host_init(int size, int rank, int device, sdns_allgather_fn fn, sdns_group_fn gfn,
                        void* user, sdns_comm** out) {
  return guarded([&] { *out = new sdns_comm{make_host_comm(size, rank, device, fn, gfn, user)}; });
}

int sdns_comm_rank(const sdns_comm* c) { return c->c->rank(); }
int sdns_comm_size(const sdns_comm* c) { return c->c->size(); }
int sdns_comm_barrier(sdns_comm* c) {
  return guarded([&] { c->c->barrier(); });
}
int sdns_comm_allreduce(sdns_comm* c, double* v, int n, int op) {
  return guarded([&] {
    if (op < 0 || op > 2) config_error("allreduce: unknown op");
    c->c->allreduce(v, n, op);
  });
}
int sdns_comm_broadcast_bytes(sdns_comm* c, void* data, int64_t nbytes, int root) {
  return guarded([&] {
    if (nbytes < 0) config_error("broadcast: negative size");
    if (nbytes && !data) config_error("broadcast: NULL buffer");
    c->c->broadcast(data, static_cast<size_t>(nbytes), root);
  });
}
int sdns_comm_destroy(sdns_comm* c) {
  return guarded([&] { delete c; });
}
int sdns_comm_poison(sdns_comm* c, const char* reason) {
  return guarded([&] { c->c->poison(reason ? reason : "poisoned"); });
}
int sdns_comm_set_timeout(sdns_comm* c, double seconds) {
  return guarded([&] { c->c->set_timeout(seconds); });
}
int sdns_comm_split(sdns_comm* c, int color, int key, sdns_comm** out) {
  return guarded([&] { *out = new sdns_comm{c->c->split(color, key)}; });
}
int sdns_comm_all_to_all_bytes(sdns_comm* c, const void* send, const int64_t* send_bytes,
                               void* recv, const int64_t* recv_bytes, void* stream) {
  return guarded([&] {
    const int p = c->c->size();
    std::vector<Xfer> xs;
    int64_t so = 0, ro = 0;
    for (int q = 0; q < p; ++q) {
      if (send_bytes[q] < 0 || recv_bytes[q] < 0) protocol_error("all_to_all: negative count");
      xs.push_back({q, static_cast<const char*>(send) + so, static_cast<char*>(recv) + ro,
                    static_cast<size_t>(send_bytes[q]), static_cast<size_t>(recv_bytes[q])});
      so += send_bytes[q];
      ro += recv_bytes[q];
    }
    SDNS_CUDA(cudaSetDevice(c->c->device()));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    c->c->alltoall(xs, s);
    if (!stream) c->c->wait(s);
  });
}

int sdns_ctx_create(const sdns_config* cfg, int rank, int device, sdns_comm* comm, void* stream,
                    sdns_ctx** out) {
  return sdns_ctx_create_ex(cfg, rank, device, comm, stream, nullptr, out);
}

int sdns_ctx_create_ex(const sdns_config* cfg, int rank, int device, sdns_comm* comm,
                       void* stream, const sdns_ctx_options* opts, sdns_ctx** out) {
  return guarded([&] {
    validate(*cfg);
    if (!comm) config_error("ctx: communicator is NULL");
    if (comm->c->size() != cfg->p)
      config_error("communicator size " + std::to_string(comm->c->size()) +
                   " does not match configured p=" + std::to_string(cfg->p));
    if (comm->c->rank() != rank) config_error("communicator rank does not match layout rank");
    // power-of-two n in [4, 1024] run the tuned kernels, every other even n
    // (validate: n >= 4, even) the generic mixed-radix ones (kernels_gen.cu);
    // their z pass holds a line's six half rows and five complex lines in
    // shared memory
    if (sdns_dev::gen_z_smem(cfg->n) > 227 * 1024)
      config_error("the sm_100a path supports n <= 1024, or non-power-of-two n up to 1780, got n=" +
                   std::to_string(cfg->n));
    if (cfg->decomp == SDNS_PENCIL && cfg->p2 > sdns_dev::kMaxSeg)
      config_error("the sm_100a pencil path needs p2 <= 16");
    auto c = std::make_unique<sdns_ctx>();
    c->cfg = *cfg;
    if (opts) c->opt = *opts;
    c->lo = build_layout(*cfg, rank);
    c->device = device;
    c->world = comm->c;
    SDNS_CUDA(cudaSetDevice(device));
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      SDNS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    const long long n = cfg->n;
    const sdns_dev_layout dl = dev_layout(*cfg, c->lo);
    c->np = dl.np;
    c->pitch = dl.pitch;
    c->prow = dl.prow;
    c->spec_cs = dl.spec_cs;
    c->real_cs = dl.real_cs;
    c->norm = 1.0 / (static_cast<double>(n) * static_cast<double>(n) * static_cast<double>(n));
    c->shells = spectrum_shells(n);
    c->tw = static_cast<double2*>(dev_alloc(c.get(), sizeof(double2) * n));
    sdns_dev::make_twiddles(static_cast<int>(n), c->tw, c->stream);
    const size_t wbytes = sizeof(double2) * static_cast<size_t>(c->spec_cs) * 6;
    c->wa = static_cast<double2*>(dev_alloc(c.get(), wbytes));
    c->pencil = cfg->decomp == SDNS_PENCIL;
    if (c->pencil) {
      // collective: row group = same coord1 ordered by coord2, column group =
      // same coord2 ordered by coord1 (fft.cpp:39-40)
      c->row = c->world->split(c->lo.coord1, c->lo.coord2);
      c->col = c->world->split(c->lo.coord2, c->lo.coord1);
      c->yl = cfg->n / cfg->p2;
      const long long rows = static_cast<long long>(c->np) * c->yl;
      c->cs_c = rows * cfg->p2 * c->pitch;
      long long base = 0;
      for (int q = 0; q < cfg->p2; ++q) {
        const int b = static_cast<int>(block_size(c->lo.nf, cfg->p2, q));
        c->seg_b.push_back(b);
        c->seg_k0.push_back(static_cast<int>(block_start(c->lo.nf, cfg->p2, q)));
        c->seg_pitch.push_back((b + 7) / 8 * 8);
        c->seg_base.push_back(base);
        base += rows * c->seg_pitch.back();
      }
      c->cs_d = base;
      c->wb = static_cast<double2*>(dev_alloc(c.get(), wbytes));
      c->map_peer_blocks(c->col.get(), cfg->p1);
      c->wc = static_cast<double2*>(dev_alloc(c.get(), sizeof(double2) * static_cast<size_t>(c->cs_c) * 6));
      c->wd = static_cast<double2*>(dev_alloc(c.get(), sizeof(double2) * static_cast<size_t>(c->cs_d) * 6));
      c->map_row_peers();
    } else {
      c->wb = cfg->p == 1 ? c->wa : static_cast<double2*>(dev_alloc(c.get(), wbytes));
      c->map_peer_blocks(c->world.get(), cfg->p);
      if (cfg->p > 1 && !c->peer && !c->opt.serial) {
        SDNS_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (auto& e : c->xev) SDNS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      // (not at 1024^3: a p = 1 RK4 state + work then needs ~157 GB without it)
      if (cfg->p == 1 && n <= 512 && is_pow2(n) && !c->opt.plain_layout) {
        c->cs_x = static_cast<long long>(c->pitch) * c->lo.spec_shape[1] * n;
        c->wx = static_cast<double2*>(dev_alloc(c.get(), sizeof(double2) * c->cs_x * 5));
        c->zchunk = n == 512;  // measured at 512
      }
      c->cmx = cfg->p == 1 && n == 1024 && !c->opt.plain_layout;
    }
    const int stride = c->shells + 3;
    const int nblk = std::max<int>(static_cast<int>(c->lo.spec_shape[0]), 592);
    c->d_partial = static_cast<double*>(dev_alloc(c.get(), sizeof(double) * stride * nblk));
    c->d_fpartial = static_cast<double*>(dev_alloc(c.get(), sizeof(double) * stride * nblk));
    c->d_fout = static_cast<double*>(dev_alloc(c.get(), sizeof(double) * stride));
    c->d_dts = static_cast<double*>(dev_alloc(c.get(), sizeof(double) * 4));
    c->d_out = static_cast<double*>(dev_alloc(c.get(), sizeof(double) * stride));
    c->d_flag = static_cast<int*>(dev_alloc(c.get(), sizeof(int)));
    SDNS_CUDA(cudaMallocHost(&c->h_out, sizeof(double) * stride));
    SDNS_CUDA(cudaMallocHost(&c->h_fout, sizeof(double) * stride));
    SDNS_CUDA(cudaMallocHost(&c->h_flag, sizeof(int)));
    c->wait();
    post_launch("ctx create");
    *out = c.release();
  });
}

int sdns_ctx_destroy(sdns_ctx* c) {
  return guarded([&] { delete c; });  // ~sdns_ctx releases everything
}

int sdns_ctx_layout(const sdns_ctx* c, sdns_layout* out) {
  *out = c->lo;
  return SDNS_OK;
}
void* sdns_ctx_stream(const sdns_ctx* c) { return c->stream; }
int sdns_ctx_transposes(const sdns_ctx* c) { return (c->peer ? 1 : 0) | (c->peer_row ? 2 : 0); }

int sdns_ctx_sync(sdns_ctx* c) {
  return guarded([&] {
    set_device(c);
    c->wait();
  });
}
int64_t sdns_ctx_device_bytes(const sdns_ctx* c) { return c->dev_bytes; }

int sdns_field_alloc(sdns_ctx* c, int kind, int ncomp, sdns_field** out) {
  return guarded([&] {
    if (ncomp < 1) config_error("field: ncomp must be >= 1");
    if (kind != SDNS_REAL && kind != SDNS_SPECTRAL) config_error("field: unknown kind");
    set_device(c);
    auto f = std::make_unique<sdns_field>();
    f->ctx = c;
    f->kind = kind;
    f->ncomp = ncomp;
    const size_t bytes = kind == SDNS_REAL ? sizeof(double) * c->real_cs * ncomp
                                           : sizeof(double2) * c->spec_cs * ncomp;
    SDNS_CUDA(cudaMalloc(&f->data, bytes));
    SDNS_CUDA(cudaMemsetAsync(f->data, 0, bytes, c->stream));
    *out = f.release();
  });
}

int sdns_field_free(sdns_field* f) {
  return guarded([&] {
    if (!f) return;
    if (f->owned) {
      cudaSetDevice(f->ctx->device);
      cudaFree(f->data);
    }
    delete f;
  });
}

int sdns_field_upload(sdns_ctx* c, sdns_field* f, const double* host) {
  return guarded([&] {
    set_device(c);
    if (f->kind == SDNS_REAL) {
      SDNS_CUDA(cudaMemcpyAsync(f->data, host, sizeof(double) * c->real_cs * f->ncomp,
                                cudaMemcpyHostToDevice, c->stream));
    } else {
      c->copy_spec_all(f->spec(), const_cast<double*>(host), f->ncomp, true);
    }
    c->wait();
  });
}

int sdns_field_download(sdns_ctx* c, const sdns_field* f, double* host) {
  return guarded([&] {
    set_device(c);
    if (f->kind == SDNS_REAL) {
      SDNS_CUDA(cudaMemcpyAsync(host, f->data, sizeof(double) * c->real_cs * f->ncomp,
                                cudaMemcpyDeviceToHost, c->stream));
    } else {
      c->copy_spec_all(f->spec(), host, f->ncomp, false);
    }
    c->wait();
  });
}

int sdns_field_copy(sdns_ctx* c, const sdns_field* src, sdns_field* dst) {
  return guarded([&] {
    if (src->kind != dst->kind || src->ncomp != dst->ncomp) config_error("field copy: shape mismatch");
    set_device(c);
    const size_t bytes = src->kind == SDNS_REAL ? sizeof(double) * c->real_cs * src->ncomp
                                                : sizeof(double2) * c->spec_cs * src->ncomp;
    SDNS_CUDA(cudaMemcpyAsync(dst->data, src->data, bytes, cudaMemcpyDeviceToDevice, c->stream));
  });
}

int sdns_fft_forward(sdns_ctx* c, const sdns_field* real, sdns_field* spec) {
  return guarded([&] {
    require_real(real, 1, "forward");
    require_spec(spec, real->ncomp, "forward");
    if (real->ncomp > 6) config_error("forward: at most 6 components per call");
    set_device(c);
    fft_forward_impl(c, real, spec);
  });
}

int sdns_fft_inverse(sdns_ctx* c, const sdns_field* spec, sdns_field* real) {
  return guarded([&] {
    require_spec(spec, 1, "inverse");
    require_real(real, spec->ncomp, "inverse");
    if (spec->ncomp > 6) config_error("inverse: at most 6 components per call");
    set_device(c);
    fft_inverse_impl(c, spec, real);
  });
}

int sdns_curl_hat(sdns_ctx* c, const sdns_field* u, sdns_field* w) {
  return guarded([&] {
    require_spec(u, 3, "curl_hat");
    require_spec(w, 3, "curl_hat");
    set_device(c);
    sdns_dev::pw_curl(u->spec(), w->spec(), c->sgeom(), c->stream);
    post_launch("curl_hat");
  });
}

int sdns_cross(sdns_ctx* c, const sdns_field* a, const sdns_field* b, sdns_field* o) {
  return guarded([&] {
    require_real(a, 3, "cross");
    require_real(b, 3, "cross");
    require_real(o, 3, "cross");
    set_device(c);
    sdns_dev::pw_cross(a->real(), b->real(), o->real(), c->real_cs, c->real_cs, c->stream);
    post_launch("cross");
  });
}

int sdns_project(sdns_ctx* c, sdns_field* u) {
  return guarded([&] {
    require_spec(u, 3, "project");
    set_device(c);
    sdns_dev::pw_project(u->spec(), c->sgeom(), c->stream);
    post_launch("project");
  });
}

int sdns_pressure_hat(sdns_ctx* c, const sdns_field* nl, sdns_field* p) {
  return guarded([&] {
    require_spec(nl, 3, "pressure_hat");
    require_spec(p, 1, "pressure_hat");
    set_device(c);
    sdns_dev::pw_pressure(nl->spec(), p->spec(), c->sgeom(), c->stream);
    post_launch("pressure_hat");
  });
}

int sdns_compute_rhs(sdns_ctx* c, const sdns_field* u, double nu, sdns_field* du) {
  return guarded([&] {
    require_spec(u, 3, "compute_rhs");
    require_spec(du, 3, "compute_rhs");
    if (u->data == du->data) config_error("compute_rhs: u_hat and du_hat must not alias");
    set_device(c);
    XfArgs a{};
    a.u = u->spec();
    a.out = du->spec();
    a.nu = nu;
    rhs_pipeline(c, u->spec(), sdns_dev::XF_TAIL, a);
  });
}

int sdns_state_create(sdns_ctx* c, sdns_state** out) {
  return guarded([&] {
    set_device(c);
    auto st = std::make_unique<sdns_state>();
    st->ctx = c;
    st->u.ctx = c;
    st->u.kind = SDNS_SPECTRAL;
    st->u.ncomp = 3;
    st->u.owned = false;
    const size_t bytes = sizeof(double2) * static_cast<size_t>(c->spec_cs) * 3;
    st->u.data = dev_alloc(c, bytes);
    st->nxt = static_cast<double2*>(dev_alloc(c, bytes));
    st->accum = static_cast<double2*>(dev_alloc(c, bytes));
    st->carry = static_cast<double2*>(dev_alloc(c, bytes));
    *out = st.release();
  });
}

int sdns_state_destroy(sdns_state* st) {
  return guarded([&] {
    if (!st) return;
    cudaSetDevice(st->ctx->device);
    cudaStreamSynchronize(st->ctx->stream);
    for (auto& g : st->ctx->graphs)  // captured steps bake this state's buffers in
      if (g.st == st && g.exec) {
        cudaGraphExecDestroy(g.exec);
        g = sdns_ctx::StepGraph{};
      }
    cudaFree(st->u.data);
    cudaFree(st->nxt);
    cudaFree(st->accum);
    cudaFree(st->carry);
    delete st;
  });
}

int sdns_state_set(sdns_ctx* c, sdns_state* st, const sdns_field* u, double t, int64_t step) {
  return guarded([&] {
    require_spec(u, 3, "state_set");
    set_device(c);
    const size_t bytes = sizeof(double2) * static_cast<size_t>(c->spec_cs) * 3;
    SDNS_CUDA(cudaMemcpyAsync(st->u.data, u->data, bytes, cudaMemcpyDeviceToDevice, c->stream));
    SDNS_CUDA(cudaMemsetAsync(st->carry, 0, bytes, c->stream));
    st->t = t;
    st->step = step;
  });
}

int sdns_state_get(sdns_ctx* c, const sdns_state* st, sdns_field* u) {
  return guarded([&] {
    require_spec(u, 3, "state_get");
    set_device(c);
    const size_t bytes = sizeof(double2) * static_cast<size_t>(c->spec_cs) * 3;
    SDNS_CUDA(cudaMemcpyAsync(u->data, st->u.data, bytes, cudaMemcpyDeviceToDevice, c->stream));
  });
}

sdns_field* sdns_state_u_hat(sdns_state* st) { return &st->u; }

int sdns_state_time(const sdns_state* st, double* t, int64_t* step) {
  if (t) *t = st->t;
  if (step) *step = st->step;
  return SDNS_OK;
}

int sdns_rk4_step(sdns_ctx* c, sdns_state* st, double dt, int post_project, int* finite) {
  return guarded([&] {
    set_device(c);
    const bool ok = step_impl(c, st, dt, post_project, finite != nullptr);
    if (finite) *finite = ok ? 1 : 0;
  });
}

int sdns_advance_hooks_run(sdns_ctx* c, sdns_state* st, const sdns_advance_hooks* hooks,
                           int64_t* fail_step) {
  return guarded([&] {
    set_device(c);
    const sdns_sample_fn sample = hooks ? hooks->sample : nullptr;
    const sdns_timing_fn timing = hooks ? hooks->timing : nullptr;
    void* user = hooks ? hooks->user : nullptr;
    const sdns_config& cfg = c->cfg;
    const int64_t n_steps = step_count(cfg.t_end, cfg.dt);
    if (sample) sample(0, st->t, user);
    for (int64_t k = 1; k <= n_steps; ++k) {
      const bool last = k == n_steps;
      const double target = last ? cfg.t_end : static_cast<double>(k) * cfg.dt;
      const double dt = target - st->t;
      const bool samp = sample && (k % cfg.out_every == 0 || last);
      const auto t0 = std::chrono::steady_clock::now();
      // a sampled step accumulates the diagnostics of its final state in the
      // last update (collect_stats of st->u inside the hook reads them); the
      // finite flag is collective and synchronises the stream
      const bool ok = step_impl(c, st, dt, 1, true, samp);
      const auto t1 = std::chrono::steady_clock::now();
      st->t = target;
      if (!ok) {
        if (fail_step) *fail_step = k;
        throw Error(SDNS_DIVERGENCE_ERROR,
                    "non-finite values in solution update at step " + std::to_string(k));
      }
      if (timing) timing(k, std::chrono::duration<double>(t1 - t0).count(), user);
      if (samp) {
        c->fused_u = &st->u;
        struct Clear {
          sdns_ctx* c;
          ~Clear() {
            c->fused_u = nullptr;
            c->fused_on_host = false;
          }
        } clear{c};
        sample(k, st->t, user);
      }
    }
  });
}

int sdns_advance(sdns_ctx* c, sdns_state* st, sdns_sample_fn sample, void* user, int64_t* fail_step) {
  const sdns_advance_hooks h{sample, nullptr, user};
  return sdns_advance_hooks_run(c, st, &h, fail_step);
}

int sdns_rk4_step_host(sdns_ctx* c, sdns_state* st, double* host, double dt, int steps) {
  return guarded([&] {
    set_device(c);
    c->copy_spec_all(st->u.spec(), host, 3, true);
    for (int k = 0; k < steps; ++k) step_impl(c, st, dt, 1, false);
    c->copy_spec_all(st->u.spec(), host, 3, false);
    c->wait();
  });
}

int sdns_collect_stats(sdns_ctx* c, const sdns_field* u, double nu, double t, double* row) {
  return guarded([&] {
    require_spec(u, 3, "collect_stats");
    set_device(c);
    stats_impl(c, u, nu, t, row);
  });
}

int sdns_l2_diff(sdns_ctx* c, const sdns_field* a, const sdns_field* b, double* out) {
  return guarded([&] {
    require_real(a, 1, "l2_diff");
    require_real(b, a->ncomp, "l2_diff");
    set_device(c);
    sdns_dev::l2_local(a->real(), b->real(), c->real_cs * a->ncomp, c->d_partial, c->d_out, c->stream);
    post_launch("l2_diff");
    SDNS_CUDA(cudaMemcpyAsync(c->h_out, c->d_out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    c->wait();
    double v = c->h_out[0];
    c->world->allreduce(&v, 1, 0);
    const double n3 = static_cast<double>(c->cfg.n) * c->cfg.n * c->cfg.n;
    *out = std::sqrt(v / n3);
  });
}

int sdns_checkpoint_write(sdns_ctx* c, const sdns_field* u, const char* path, double t,
                          int64_t step) {
  return guarded([&] {
    require_real(u, 3, "write_checkpoint");
    set_device(c);
    c->wait();
    checkpoint_write_impl(c, u, path ? path : "", t, step);
  });
}

int sdns_checkpoint_read(sdns_ctx* c, const char* path, sdns_field* u, double* t, int64_t* step) {
  return guarded([&] {
    require_real(u, 3, "read_checkpoint");
    set_device(c);
    c->wait();
    checkpoint_read_impl(c, path ? path : "", u, t, step);
  });
}

int sdns_ctx_timing(sdns_ctx* c, int enable) {
  return guarded([&] {
    set_device(c);
    if (enable && c->ev.empty()) {
      const size_t nev = 16384;
      c->ev.resize(nev);
      c->ev_tag.assign(nev, 0);
      for (auto& e : c->ev) SDNS_CUDA(cudaEventCreate(&e));
    }
    c->timing = enable != 0;
    c->ev_used = 0;
  });
}

int sdns_ctx_timing_read(sdns_ctx* c, double* ms, int64_t* launches) {
  return guarded([&] {
    set_device(c);
    c->wait();
    for (int t = 0; t < SDNS_NPASS; ++t) {
      ms[t] = 0.0;
      launches[t] = 0;
    }
    for (size_t i = 0; i + 1 < c->ev_used + 1 && i < c->ev_used; i += 2) {
      float f = 0.0f;
      SDNS_CUDA(cudaEventElapsedTime(&f, c->ev[i], c->ev[i + 1]));
      const int t = c->ev_tag[i];
      ms[t] += static_cast<double>(f);
      launches[t] += 1;
    }
    c->ev_used = 0;
  });
}

void* sdns_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}
void sdns_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
