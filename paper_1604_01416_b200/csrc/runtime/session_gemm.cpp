// One worker's K-panel pipeline of one distributed GEMM command -- the B200
// form of GeneralGemmExec / CyclicGemmExec / CachedBackwardExec's
// "assemble op(A) rows and op(B) columns, then local_gemm" (ops.hpp:214-330,
// 336-383, 406-503): the same pieces, pulled panel by panel and overlapped
// with the tcgen05 GEMM.
//
// Consumer-split schedule, per panel step s (panels in `order`, the
// least-remote first):
//   pull   (stream `pull`, copy engines): pieces on another GPU land in a
//          double-buffered local buffer; a stream memory op then publishes
//          the step's sequence number in the worker's flag word;
//   split  (stream `side`, or -- tf32 / mixed planes, when it pays -- the
//          split warps of step s-1's GEMM launches): transpose/assemble into
//          K-major planes (scaled fp16 pair, or tf32 hi + tf32 lo / bf16 hi, lo);
//   GEMM   (stream `stream`): C += op(A)_s op(B)_s over double-buffered planes.
// Buffer reuse is event-ordered: landing[s % 2] waits until step s-2's split
// consumed it, planes[s % 2] until step s-2's GEMM read them.
// Presplit schedule (run_presplit): no split here -- the owners split their
// blocks (session_presplit.cpp); per step the pull stream copies plane
// rectangles and row maxima from the owners' arenas into planes[s % 2] (or
// the step reads a wholly-local panel in place), then the GEMM.
#include <algorithm>
#include <array>
#include <cstring>
#include <deque>
#include <functional>
#include <map>

#include "../kernels/tf32x3_gemm.h"
#include "session.hpp"

namespace dm {

struct Session::GemmRun {
  // panel planes of one range and buffer: fp32 hi, and either fp32 lo
  // (tf32x3) or bf16 hi + bf16 lo packed in one buffer (mixed); 8 B/element.
  // K-major [len x kpitch] when the range's pieces are stored row-wise along
  // K; MN-major [kpitch x ld] (ld = len rounded to 32) when they are stored
  // K-row-wise (a transposed A, a non-transposed B), so every split reads its
  // source row by row and none transposes.
  // kModeF16x2: hi = lo = null, hi16 / lo16 = fp16 h0 / h1 (4 B / element
  // together), rmax = the rows' |x| maxima (their power-of-two scales).
  struct Planes {
    float* hi;
    float* lo;
    void* hi16;
    void* lo16;
    bool mn;
    std::int64_t ld;  // pitch of every plane (elements)
    unsigned* rmax = nullptr;
  };
  // one split item per piece: effective source (the landing buffer for pieces
  // that crossed a link), target planes, and whether it waits on the flag
  struct Item {
    const void* src;
    std::int64_t lds;
    const Piece* pc;
    const Planes* pl;
    bool landed;
    cudaEvent_t ready;  // landed chunk: its own copy-done event (separate splits wait on it)
  };

  Session& S;
  Worker& w;
  const GemmArgs& g;
  const SourcePolicy pol;
  const WorkerPlan plan;
  std::vector<DeviceBuffer>& bufs;
  std::vector<cudaEvent_t>& events;

  // command-wide settings
  const bool half_in;  // Half16 operands: fp32 compute, C rounded once (AccumOf<Half>, kernels.hpp:29-35)
  const std::size_t esz;
  const int gemm_mode;
  const bool trace;
  const bool presplit;  // planes come split from their owners' plane arenas (session_presplit.cpp)
  const int np;
  const int nbuf;
  std::int64_t kpitch = 8;
  int lockstep = 0;
  bool exclusive = true;  // this worker's GEMMs have the device to themselves (co-resident CTAs)
  std::int64_t fuse_mode = 1;
  unsigned* phase_ctr = nullptr;  // kModeF16x2 fused splits: one grid-handoff counter per step

  std::vector<std::array<Planes, 2>> pa, pb;
  std::vector<std::vector<Planes>> spa, spb;  // presplit: per step, per range (an arena alias or pa / pb)
  std::vector<int> order;
  bool use_ce = false;
  char* landing[2] = {nullptr, nullptr};
  unsigned* flag = nullptr;
  std::vector<cudaEvent_t> landed_ev, consumed_ev, split_ev, gemm_ev;
  std::vector<std::vector<Item>> items;
  std::deque<Piece> chunk_pieces;  // sub-pieces of chunked pulls (stable addresses)
  std::map<BlockKey, std::uint64_t> pulled_blocks;  // remote bytes read per block (trace())
  std::vector<unsigned> seq;
  unsigned* sync = nullptr;  // lockstep counters
  std::size_t sync_bytes = 0;
  float* ksplit_ws = nullptr;  // split-K partials (stream-ordered reuse)
  std::size_t ksplit_ws_bytes = 0;

  GemmRun(Session& s, Worker& wk, const GemmArgs& ga, SourcePolicy p, WorkerPlan pl, std::vector<DeviceBuffer>& b,
          std::vector<cudaEvent_t>& e, bool presplit_cmd = false)
      : S(s), w(wk), g(ga), pol(p), plan(std::move(pl)), bufs(b), events(e),
        half_in(s.table_.at(ga.a).precision == Precision::Half16),
        esz(byte_width(s.table_.at(ga.a).precision)),
        gemm_mode(split_mode_for(s.gemm_mode_, plan.k0.empty() ? 0 : plan.k0.back(), half_in, work_of(s, ga, plan))),
        trace(s.tracing() && !s.async_),
        presplit(presplit_cmd),
        np(static_cast<int>(plan.k0.size()) - 1),
        nbuf(np > 1 ? 2 : 1) {
    std::int64_t kmax = 0;
    for (int p = 0; p < np; ++p) kmax = std::max(kmax, plan.k0[p + 1] - plan.k0[p]);
    kpitch = std::max<std::int64_t>(8, (kmax + 7) / 8 * 8);
  }

  // Half16 operands are exact in one tf32 term: they keep 3xTF32 (their
  // splits read fp16 sources, which the scaled fp16 pair does not take).
  static int split_mode_for(int session_mode, std::int64_t k, bool half, double work) {
    const int m = resolve_split_mode(session_mode, k, work);
    return half && m == kModeF16x2 ? kModeTf32x3 : m;
  }
  bool f16x2() const { return gemm_mode == kModeF16x2; }
  // 2 m n K over this worker's C blocks
  static double work_of(const Session& s, const GemmArgs& g, const WorkerPlan& p) {
    double work = 0;
    const BlockGrid& gc = s.table_.at(g.c).layout.grid;
    for (const Task& t : p.tasks) {
      auto [mb, nb] = block_extent(gc, t.c);
      work += 2.0 * mb * nb * static_cast<double>(p.k0.empty() ? 0 : p.k0.back());
    }
    return work;
  }

  cudaEvent_t new_event() {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    events.push_back(e);
    return e;
  }

  // ------------------------------------------------------------ setup
  void setup() {
    // Producer lockstep needs the GEMM's CTAs co-resident: off when another
    // local worker shares this device (its GEMMs run concurrently).
    int sharing = 0;
    for (auto& o : S.workers_) sharing += (o && o->device == w.device) ? 1 : 0;
    exclusive = sharing == 1;
    lockstep = exclusive ? static_cast<int>(env_int("DM_LOCKSTEP", 32)) : 0;
    // DM_FUSE_SPLIT: 0 never, 1 when the carrying GEMM hides the split, 2 always.
    // Not by default for the scaled fp16 pair: its two-phase fused split slows
    // the carrying GEMM by ~4 ms per GiB (9.9 -> 13.8 ms per 8192-wide panel at
    // 4 GPUs), while its own kernels split a GiB in ~0.65 ms between the
    // GEMMs (4 GPUs: 1543 vs 1260 TFLOP/s, profiles/r02/fuse_ab/).
    fuse_mode = (half_in || presplit) ? 0 : env_int("DM_FUSE_SPLIT", f16x2() ? 0 : 1);

    alloc_planes(plan.ar, plan.br, true, pa);
    alloc_planes(plan.br, plan.ar, false, pb);
    if (f16x2() && np > 1 && !presplit) {
      bufs.push_back(w.pool->acquire(static_cast<std::size_t>(np) * 4));
      phase_ctr = static_cast<unsigned*>(bufs.back().data());
    }
    // operands of this worker's GEMMs were written by earlier commands on
    // its own streams; order the split stream after the compute stream
    cudaEvent_t e = new_event();
    cuda_check(cudaEventRecord(e, w.stream), "event");
    cuda_check(cudaStreamWaitEvent(w.side, e, 0), "wait");

    order_panels();
    if (presplit) {
      // every owner's planes (this command's owner splits, then the barrier)
      for (auto& o : S.workers_)
        if (o && o->presplit_done)
          for (cudaStream_t st : {w.pull, w.stream})
            cuda_check(cudaStreamWaitEvent(st, o->presplit_done, 0), "wait presplit");
      spa.assign(np, {});
      spb.assign(np, {});
    } else {
      setup_landing();
    }
    landed_ev.assign(np, nullptr);
    consumed_ev.assign(np, nullptr);
    split_ev.assign(np, nullptr);
    gemm_ev.assign(np, nullptr);
    items.assign(np, {});
    seq.assign(np, 0);
  }

  // MN-major planes for a range whose pieces are transposed (all pieces of a
  // range come from one operand, so they share the flag) -- when the planes
  // are reused by few output rows/columns (`reuse` = the other operand's
  // extent over this worker's tasks).  The tensor core reads MN-major tiles
  // ~10% slower (tools/micro/mn_probe.cu: 269 vs 235 TFLOP/s at 16384^3), so a
  // long GEMM prefers the transposing split (~0.4 ms/GiB extra); a short,
  // memory-bound one (FC strips) prefers the direct split.  Break-even
  // ~2000 rows (DM_MN_REUSE).
  static bool range_mn(const Range& r, std::int64_t reuse) {
    if (reuse >= env_int("DM_MN_REUSE", 2048)) return false;  // (f16x2 planes are always K-major)
    for (const auto& panel : r.panels)
      for (const Piece& pc : panel) return pc.trans != 0;
    return false;
  }

  struct PlaneShape {
    bool mn;
    std::int64_t ld;
    std::size_t elems;
  };
  PlaneShape plane_shape(const std::vector<Range>& rs, const std::vector<Range>& other, bool is_a,
                         std::size_t i) const {
    std::int64_t reuse = 0;
    for (const Task& t : plan.tasks)
      if ((is_a ? t.ra : t.rb) == static_cast<int>(i)) reuse += other[is_a ? t.rb : t.ra].len;
    const bool mn = !f16x2() && range_mn(rs[i], reuse);
    const std::int64_t len = std::max<std::int64_t>(rs[i].len, 1);
    const std::int64_t ld = mn ? (len + 31) / 32 * 32 : kpitch;
    return {mn, ld, static_cast<std::size_t>(mn ? kpitch * ld : len * kpitch)};
  }

  // Plane-cache key of A range i (GemmArgs::plane_cache_a, single panel):
  // everything the split planes' content and layout depend on but A's version.
  bool plane_cacheable() const { return g.plane_cache_a && np == 1 && !half_in; }
  std::vector<std::int64_t> plane_key(std::size_t i) const {
    const PlaneShape sh = plane_shape(plan.ar, plan.br, true, i);
    return {static_cast<std::int64_t>(g.a), g.trans_a ? 1 : 0, plan.ar[i].start, plan.ar[i].len, plan.k0.back(),
            sh.mn ? 1 : 0, sh.ld, gemm_mode};
  }
  // Cached A planes of range i: the entry (or null) and whether it holds A's
  // current version (its split can then be skipped).
  Worker::PlaneCache* plane_entry(std::size_t i, bool* fresh) const {
    *fresh = false;
    if (!plane_cacheable()) return nullptr;
    auto it = w.plane_cache.find(plane_key(i));
    if (it == w.plane_cache.end()) return nullptr;
    *fresh = it->second.filled && it->second.version == S.table_.at(g.a).version;
    return &it->second;
  }
  std::vector<char> a_fresh;  // per A range: planes served by the plane cache

  void alloc_planes(const std::vector<Range>& rs, const std::vector<Range>& other, bool is_a,
                    std::vector<std::array<Planes, 2>>& out) {
    out.resize(rs.size());
    if (is_a) a_fresh.assign(rs.size(), 0);
    for (std::size_t i = 0; i < rs.size(); ++i) {
      const PlaneShape sh = plane_shape(rs, other, is_a, i);
      const std::size_t rmax_bytes = static_cast<std::size_t>(std::max<std::int64_t>(rs[i].len, 1)) * 4;
      for (int b = 0; b < nbuf; ++b) {
        float* hi;
        char* second;
        unsigned* rmax = nullptr;
        if (is_a && plane_cacheable()) {
          Worker::PlaneCache& pc = w.plane_cache[plane_key(i)];
          if (!pc.hi.data()) {
            pc.hi = w.pool->acquire(sh.elems * 4);
            if (f16x2()) pc.rmax = w.pool->acquire(rmax_bytes);
            else pc.second = w.pool->acquire(sh.elems * 4);
          }
          a_fresh[i] = pc.filled && pc.version == S.table_.at(g.a).version ? 1 : 0;
          hi = pc.hi.f32();
          second = static_cast<char*>(pc.second.data());
          rmax = static_cast<unsigned*>(pc.rmax.data());
        } else {
          bufs.push_back(w.pool->acquire(sh.elems * 4));
          hi = bufs.back().f32();
          if (f16x2()) {
            bufs.push_back(w.pool->acquire(rmax_bytes));
            rmax = static_cast<unsigned*>(bufs.back().data());
            second = nullptr;
          } else {
            bufs.push_back(w.pool->acquire(sh.elems * 4));
            second = static_cast<char*>(bufs.back().data());
          }
        }
        if (f16x2()) {
          char* h = reinterpret_cast<char*>(hi);  // fp16 h0 | h1, sh.elems each
          out[i][b] = Planes{nullptr, nullptr, h, h + sh.elems * 2, false, sh.ld, rmax};
        } else {
          out[i][b] = gemm_mode == kModeMixed
                          ? Planes{hi, nullptr, second, second + sh.elems * 2, sh.mn, sh.ld}
                          : Planes{hi, reinterpret_cast<float*>(second), nullptr, nullptr, sh.mn, sh.ld};
        }
      }
    }
  }

  // After this command's splits are enqueued (or its graph launched): the
  // cached A planes hold A's current version.
  void commit_plane_cache() {
    if (!plane_cacheable()) return;
    for (std::size_t i = 0; i < plan.ar.size(); ++i) {
      auto it = w.plane_cache.find(plane_key(i));
      if (it != w.plane_cache.end()) {
        it->second.version = S.table_.at(g.a).version;
        it->second.filled = true;
      }
    }
  }

  // Everything the captured launches of this command depend on (graph key):
  // the command, the operand pieces' source pointers, the C blocks, the
  // plane-cache state, the split scheme and the tuning knobs read while issuing.
  std::vector<std::uint64_t> signature() const {
    std::vector<std::uint64_t> sig;
    auto put = [&](std::uint64_t v) { sig.push_back(v); };
    auto putd = [&](double d) {
      std::uint64_t u;
      std::memcpy(&u, &d, 8);
      put(u);
    };
    put(static_cast<std::uint64_t>(pol));
    put(g.a);
    put(g.b);
    put(g.c);
    put((g.trans_a ? 1u : 0u) | (g.trans_b ? 2u : 0u) | (g.plane_cache_a ? 4u : 0u));
    putd(g.alpha);
    putd(g.beta);
    put(static_cast<std::uint64_t>(gemm_mode));
    put(static_cast<std::uint64_t>(np));
    static const char* knobs[] = {"DM_FUSE_SPLIT", "DM_CTA_GROUP", "DM_FLUSH_K", "DM_GROUP_M", "DM_L2_POLICY",
                                  "DM_LOCKSTEP", "DM_MN_REUSE", "DM_PULL_CE", "DM_SPLIT_WARPS", "DM_C_PREFETCH",
                                  "DM_KSPLIT"};
    for (const char* k : knobs) {
      const char* v = std::getenv(k);
      put(v ? std::hash<std::string>()(v) : 0);
    }
    for (const auto* ranges : {&plan.ar, &plan.br})
      for (const Range& r : *ranges) {
        put(static_cast<std::uint64_t>(r.start));
        put(static_cast<std::uint64_t>(r.len));
        for (const auto& panel : r.panels)
          for (const Piece& pc : panel) {
            bool remote = false;
            put(reinterpret_cast<std::uintptr_t>(S.source_ptr(w, pc.matrix, pc.coord, pol, &remote)));
            put(static_cast<std::uint64_t>(pc.src_off) * 2 + (remote ? 1 : 0));
          }
      }
    for (const Task& t : plan.tasks) put(reinterpret_cast<std::uintptr_t>(w.owned.at({g.c, t.c}).mem.data()));
    for (std::size_t i = 0; i < plan.ar.size(); ++i) {
      bool fresh = false;
      const Worker::PlaneCache* pc = plane_entry(i, &fresh);
      put(pc ? reinterpret_cast<std::uintptr_t>(pc->hi.data()) * 2 + (fresh ? 1 : 0) : 0);
    }
    return sig;
  }

  template <class F>
  void for_pieces(int p, F&& f) const {
    for (const auto* ranges : {&plan.ar, &plan.br})
      for (const Range& r : *ranges)
        for (const Piece& pc : r.panels[p]) f(pc);
  }

  // Panels with the fewest peer bytes first: the GEMM starts on local data
  // while the first remote pulls are in flight (K order does not matter
  // mathematically; every panel accumulates into C).
  void order_panels() {
    order.resize(np);
    for (int p = 0; p < np; ++p) order[p] = p;
    if (np < 2) return;
    std::vector<std::uint64_t> remote_bytes(np, 0);
    for (int p = 0; p < np; ++p)
      for_pieces(p, [&](const Piece& pc) {
        bool remote = false;
        S.source_ptr(w, pc.matrix, pc.coord, pol, &remote);
        if (remote) remote_bytes[p] += pc.bytes();
      });
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return remote_bytes[x] < remote_bytes[y]; });
  }

  // Copy engines carry remote pieces only when panels pipeline: there the
  // transfer must not take SMs from the concurrently running GEMM.  A
  // single-panel command has nothing to overlap, and one split kernel that
  // reads peer memory directly moves the bytes once instead of twice.
  const void* resolve(const Piece& pc, bool* remote, bool* cross) const {
    const void* src = static_cast<const char*>(S.source_ptr(w, pc.matrix, pc.coord, pol, remote)) +
                      pc.src_off * static_cast<std::int64_t>(esz);
    *cross = false;
    if (*remote && use_ce) {
      const Worker* ow = S.local(S.table_.at(pc.matrix).layout.owner(pc.coord));
      *cross = ow == nullptr || ow->device != w.device;
    }
    return src;
  }
  // landing rectangle of a piece: source rows (op-k rows when transposed)
  static std::int64_t land_width(const Piece& pc) { return pc.trans ? pc.rows : pc.kcols; }
  static std::int64_t land_height(const Piece& pc) { return pc.trans ? pc.kcols : pc.rows; }
  static std::int64_t land_pitch(const Piece& pc) { return (land_width(pc) + 7) / 8 * 8; }
  std::size_t land_bytes(const Piece& pc) const {
    return static_cast<std::size_t>((land_pitch(pc) * land_height(pc) * static_cast<std::int64_t>(esz) + 255) /
                                    256 * 256);
  }

  void setup_landing() {
    use_ce = env_int("DM_PULL_CE", 1) != 0 && np > 1;
    std::size_t land_max = 0;
    for (int p = 0; p < np; ++p) {
      std::size_t tot = 0;
      for_pieces(p, [&](const Piece& pc) {
        bool remote, cross;
        resolve(pc, &remote, &cross);
        if (cross) tot += land_bytes(pc);
      });
      land_max = std::max(land_max, tot);
    }
    if (land_max == 0) return;
    for (int b = 0; b < nbuf; ++b) {
      bufs.push_back(w.pool->acquire(land_max));
      landing[b] = static_cast<char*>(bufs.back().data());
    }
    if (!w.pull_flag.data()) {
      w.pull_flag = w.pool->acquire(256);
      cuda_check(cudaMemset(w.pull_flag.data(), 0, 256), "cudaMemset(flag)");
      w.pull_seq = 0;
    }
    flag = static_cast<unsigned*>(w.pull_flag.data());
    // the copy stream starts where the split stream is (after the operand
    // waits / device barrier of the command)
    cudaEvent_t e = new_event();
    cuda_check(cudaEventRecord(e, w.side), "event");
    cuda_check(cudaStreamWaitEvent(w.pull, e, 0), "wait");
  }

  // ------------------------------------------------------------ per step
  // Issue the copy-engine pulls of step s and build its split items.
  void prepare(int s) {
    const int p = order[s];
    const int buf = s % nbuf;
    std::size_t loff = 0;
    std::uint64_t pulled = 0;
    cudaEvent_t tp = nullptr;
    bool any = false;
    for (int ab = 0; ab < 2; ++ab) {
      const std::vector<Range>& rs = ab == 0 ? plan.ar : plan.br;
      const std::vector<std::array<Planes, 2>>& planes = ab == 0 ? pa : pb;
      for (std::size_t i = 0; i < rs.size(); ++i) {
        if (ab == 0 && !a_fresh.empty() && a_fresh[i]) continue;  // planes already hold this version
        for (const Piece& pc : rs[i].panels[p]) {
          bool remote, cross;
          const void* src = resolve(pc, &remote, &cross);
          (remote ? w.stats.peer_bytes_read : w.stats.local_bytes_read) += pc.bytes() / 4 * esz;
          if (remote) pulled_blocks[{pc.matrix, pc.coord}] += pc.bytes() / 4 * esz;
          if (!cross) {
            items[s].push_back({src, pc.lds, &pc, &planes[i][buf], false, nullptr});
            continue;
          }
          if (!any) {
            any = true;
            // landing[buf] was last read by the split of step s - nbuf
            if (s >= nbuf) cuda_check(cudaStreamWaitEvent(w.pull, consumed_ev[s - nbuf], 0), "wait");
            if (trace) tp = S.trace_event(w.pull);
          }
          // The first panel's pull is exposed (its split runs before any
          // GEMM): cut it into row chunks of about DM_PULL_CHUNK_MB, each with
          // its own event, so splitting chunk i overlaps copying chunk i+1.
          // Later panels stay whole (their splits are usually fused).
          const std::int64_t h = land_height(pc);
          const std::int64_t chunk_mb = s == 0 ? env_int("DM_PULL_CHUNK_MB", 128) : 0;
          const std::int64_t row_bytes = land_width(pc) * static_cast<std::int64_t>(esz);
          const std::int64_t rows_per =
              chunk_mb > 0 ? std::max<std::int64_t>(8, (chunk_mb << 20) / std::max<std::int64_t>(1, row_bytes)) : h;
          const std::int64_t lp = land_pitch(pc);
          char* dst = landing[buf] + loff;
          for (std::int64_t h0 = 0; h0 < h; h0 += rows_per) {
            const std::int64_t hn = std::min(rows_per, h - h0);
            const Piece* sub = &pc;
            if (hn != h) {  // sub-piece: rows (direct) or k (transposed) [h0, h0 + hn)
              Piece q = pc;
              if (pc.trans) {
                q.kcols = hn;
                q.dst_k = pc.dst_k + h0;
              } else {
                q.rows = hn;
                q.dst_row = pc.dst_row + h0;
              }
              chunk_pieces.push_back(q);
              sub = &chunk_pieces.back();
            }
            char* cdst = dst + h0 * lp * static_cast<std::int64_t>(esz);
            const char* csrc = static_cast<const char*>(src) + h0 * pc.lds * static_cast<std::int64_t>(esz);
            cuda_check(cudaMemcpy2DAsync(cdst, lp * esz, csrc, pc.lds * esz, land_width(pc) * esz, hn,
                                         cudaMemcpyDefault, w.pull),
                       "cudaMemcpy2DAsync(peer)");
            cudaEvent_t ready = nullptr;
            if (hn != h) {
              ready = new_event();
              cuda_check(cudaEventRecord(ready, w.pull), "event");
            }
            items[s].push_back({cdst, lp, sub, &planes[i][buf], true, ready});
          }
          loff += land_bytes(pc);
          pulled += pc.bytes() / 4 * esz;
        }
      }
    }
    if (!any) return;
    landed_ev[s] = new_event();
    seq[s] = ++w.pull_seq;
    cuda_check(stream_write_flag(w.pull, flag, seq[s]), "cuStreamWriteValue32");
    cuda_check(cudaEventRecord(landed_ev[s], w.pull), "event");
    if (trace) w.trace.push_back({"pull", p, pulled, 0.0, tp, S.trace_event(w.pull)});
  }

  // ------------------------------------------------------------ presplit
  // Where piece `pc` (role 0: A, 1: B) lies in its owner's plane arena.
  struct Loc {
    const char* base;
    const ArenaBlock* ab;
    std::int64_t o, q;  // plane row and k offset inside the owner block
    int owner;
  };
  std::map<int, std::map<std::pair<int, BlockKey>, ArenaBlock>> arena_maps;
  Loc locate(int role, const Piece& pc) {
    const int owner = S.table_.at(pc.matrix).layout.owner(pc.coord);
    auto it = arena_maps.find(owner);
    if (it == arena_maps.end()) {
      std::size_t t = 0;
      it = arena_maps.emplace(owner, S.plane_arena_map(g, owner, &t)).first;
    }
    const ArenaBlock& ab = it->second.at({role, BlockKey{pc.matrix, pc.coord}});
    if (ab.trans != pc.trans) throw ProtocolError("presplit: piece orientation differs from its arena planes");
    const std::int64_t a = pc.src_off / pc.lds, b = pc.src_off % pc.lds;
    return {S.plane_arena_ptrs_.at(owner), &ab, pc.trans ? b : a, pc.trans ? a : b, owner};
  }

  // Planes of step s: a range whose panel is one whole local piece aliases
  // the owner arena (no copy); every other range gets its pieces' plane
  // rectangles and row maxima copied into its panel buffer on the copy
  // engines (peer arenas over NVLink).
  void prepare_presplit(int s) {
    const int p = order[s];
    const int buf = s % nbuf;
    bool any = false;
    cudaEvent_t tp = nullptr;
    std::uint64_t pulled = 0;
    for (int ab = 0; ab < 2; ++ab) {
      const std::vector<Range>& rs = ab == 0 ? plan.ar : plan.br;
      const std::vector<std::array<Planes, 2>>& planes = ab == 0 ? pa : pb;
      std::vector<Planes>& sp = (ab == 0 ? spa : spb)[s];
      sp.resize(rs.size());
      for (std::size_t i = 0; i < rs.size(); ++i) {
        const std::vector<Piece>& pieces = rs[i].panels[p];
        if (pieces.size() == 1) {
          const Piece& pc = pieces[0];
          const Loc L = locate(ab, pc);
          if (L.owner == w.id && pc.rows == rs[i].len && L.q % 8 == 0) {
            const std::int64_t off = (L.o * L.ab->ld + L.q) * 2;
            char* base = const_cast<char*>(L.base);
            sp[i] = Planes{nullptr, nullptr, base + L.ab->h0 + off, base + L.ab->h1 + off, false, L.ab->ld,
                           reinterpret_cast<unsigned*>(base + L.ab->grmax) + L.o};
            w.stats.local_bytes_read += pc.bytes();
            continue;
          }
        }
        const Planes& dst = planes[i][buf];
        sp[i] = dst;
        for (const Piece& pc : pieces) {
          const Loc L = locate(ab, pc);
          if (!any) {
            any = true;
            // planes[buf] was last read by the GEMM of step s - nbuf
            if (s >= nbuf) cuda_check(cudaStreamWaitEvent(w.pull, gemm_ev[s - nbuf], 0), "wait");
            if (trace) tp = S.trace_event(w.pull);
          }
          for (int h = 0; h < 2; ++h) {
            const char* src = L.base + (h ? L.ab->h1 : L.ab->h0) + (L.o * L.ab->ld + L.q) * 2;
            char* d = static_cast<char*>(h ? dst.lo16 : dst.hi16) + (pc.dst_row * dst.ld + pc.dst_k) * 2;
            cuda_check(cudaMemcpy2DAsync(d, dst.ld * 2, src, L.ab->ld * 2, pc.kcols * 2, pc.rows, cudaMemcpyDefault,
                                         w.pull),
                       "cudaMemcpy2DAsync(planes)");
          }
          if (pc.dst_k == 0)  // the row scales: once per row (every piece of a row carries the same)
            cuda_check(cudaMemcpyAsync(dst.rmax + pc.dst_row, L.base + L.ab->grmax + L.o * 4, pc.rows * 4,
                                       cudaMemcpyDefault, w.pull),
                       "cudaMemcpyAsync(row maxima)");
          if (L.owner != w.id) {
            w.stats.peer_bytes_read += pc.bytes();
            pulled_blocks[{pc.matrix, pc.coord}] += pc.bytes();
            pulled += pc.bytes();
          } else {
            w.stats.local_bytes_read += pc.bytes();
          }
        }
      }
    }
    if (!any) return;
    landed_ev[s] = new_event();
    cuda_check(cudaEventRecord(landed_ev[s], w.pull), "event");
    split_ev[s] = landed_ev[s];  // the GEMM of step s waits for its planes
    if (trace) w.trace.push_back({"pull", p, pulled, 0.0, tp, S.trace_event(w.pull)});
  }

  void run_presplit() {
    setup();
    prepare_presplit(0);
    for (int step = 0; step < np; ++step) {
      if (step + 1 < np) prepare_presplit(step + 1);
      gemm_step(step, nullptr);
    }
    // the next presplit command's owner splits wait for these reads
    if (!w.plane_reads) cuda_check(cudaEventCreateWithFlags(&w.plane_reads, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(w.plane_reads, w.stream), "event");
    log_pulls();
  }

  std::int64_t plane_off(const Item& it) const {
    return it.pl->mn ? it.pc->dst_k * it.pl->ld + it.pc->dst_row : it.pc->dst_row * it.pl->ld + it.pc->dst_k;
  }
  // split_tf32 shape of an item: x[r][q] = trans ? src[q * lds + r] : src[r * lds + q]
  // lands at plane + r * ld + q; an MN-major plane stores op(X)^T, i.e. the
  // piece with rows and columns swapped and the transpose flag flipped
  struct SplitShape {
    int trans;
    std::int64_t rows, cols;
  };
  static SplitShape split_shape(const Item& it) {
    const Piece& pc = *it.pc;
    return it.pl->mn ? SplitShape{pc.trans ? 0 : 1, pc.kcols, pc.rows} : SplitShape{pc.trans, pc.rows, pc.kcols};
  }

  // kModeF16x2: clear the row maxima the splits of step s accumulate into
  // (every range has pieces in every panel; cache-fresh A planes keep theirs).
  void zero_rmax(int s, cudaStream_t st) {
    if (!f16x2()) return;
    const int buf = s % nbuf;
    for (int ab = 0; ab < 2; ++ab) {
      const std::vector<Range>& rs = ab == 0 ? plan.ar : plan.br;
      const std::vector<std::array<Planes, 2>>& planes = ab == 0 ? pa : pb;
      for (std::size_t i = 0; i < rs.size(); ++i) {
        if (ab == 0 && !a_fresh.empty() && a_fresh[i]) continue;
        cuda_check(cudaMemsetAsync(planes[i][buf].rmax, 0, static_cast<std::size_t>(std::max<std::int64_t>(rs[i].len, 1)) * 4, st),
                   "memset row maxima");
      }
    }
  }

  // Split step s with its own kernels on the split stream.
  void split_separate(int s) {
    if (s >= nbuf) cuda_check(cudaStreamWaitEvent(w.side, gemm_ev[s - nbuf], 0), "wait");  // planes free
    zero_rmax(s, w.side);
    cudaEvent_t ta = trace ? S.trace_event(w.side) : nullptr;
    std::uint64_t bytes = 0;
    // Small splits (a latency-bound command): every piece in one launch.
    if (split_batched(s)) {
      if (trace) w.trace.push_back({"split", order[s], 0, 0.0, ta, S.trace_event(w.side)});
      split_ev[s] = new_event();
      cuda_check(cudaEventRecord(split_ev[s], w.side), "event");
      consumed_ev[s] = split_ev[s];
      return;
    }
    // local pieces first (no wait), then landed ones as their copies complete
    std::vector<const Item*> seq_items;
    for (const Item& it : items[s])
      if (!it.landed) seq_items.push_back(&it);
    for (const Item& it : items[s])
      if (it.landed) seq_items.push_back(&it);
    if (f16x2()) {
      // row maxima of every piece first (a plane row's scale spans its pieces),
      // then the splits
      for (const Item* itp : seq_items) {
        const Item& it = *itp;
        if (it.landed)
          cuda_check(cudaStreamWaitEvent(w.side, it.ready ? it.ready : landed_ev[s], 0), "wait");
        const SplitShape sh = split_shape(it);
        cuda_check(absmax_rows(static_cast<const float*>(it.src), it.lds, sh.trans, sh.rows, sh.cols,
                               it.pl->rmax + it.pc->dst_row, w.side),
                   "absmax_rows");
        w.stats.split_launches += 1;
      }
      for (const Item* itp : seq_items) {
        const Item& it = *itp;
        const Planes& pl = *it.pl;
        const std::int64_t off = plane_off(it);
        const SplitShape sh = split_shape(it);
        cuda_check(split_f16x2(static_cast<const float*>(it.src), it.lds, sh.trans, sh.rows, sh.cols,
                               static_cast<char*>(pl.hi16) + off * 2, static_cast<char*>(pl.lo16) + off * 2, pl.ld,
                               pl.rmax + it.pc->dst_row, w.side),
                   "split_f16x2");
        w.stats.split_launches += 1;
        bytes += it.pc->bytes() / 4 * esz;
      }
      seq_items.clear();
    }
    for (const Item* itp : seq_items) {
      const Item& it = *itp;
      if (it.landed)
        cuda_check(cudaStreamWaitEvent(w.side, it.ready ? it.ready : landed_ev[s], 0), "wait");
      const Piece& pc = *it.pc;
      const Planes& pl = *it.pl;
      const std::int64_t off = plane_off(it);
      const SplitShape sh = split_shape(it);
      cuda_check(split_tf32(it.src, half_in ? 1 : 0, it.lds, sh.trans, sh.rows, sh.cols, pl.hi + off,
                            pl.lo ? pl.lo + off : nullptr, pl.ld,
                            pl.hi16 ? static_cast<char*>(pl.hi16) + off * 2 : nullptr,
                            pl.lo16 ? static_cast<char*>(pl.lo16) + off * 2 : nullptr, pl.ld, w.side),
                 "split_tf32");
      w.stats.split_launches += 1;
      bytes += pc.bytes() / 4 * esz;
    }
    if (trace) w.trace.push_back({"split", order[s], bytes, 0.0, ta, S.trace_event(w.side)});
    split_ev[s] = new_event();
    cuda_check(cudaEventRecord(split_ev[s], w.side), "event");
    consumed_ev[s] = split_ev[s];
  }

  // One split_jobs launch for all items of step s when there are several,
  // they are small (<= DM_BATCH_SPLIT_MB of input, default 64) and none waits
  // on a landing.  Measured at 4 GPUs: 2048^3 on 2x2 95 -> 90 us, FC dW
  // (8 pieces) 128 -> 98 us; a single piece is faster in its own vectorised
  // kernel (FC forward: 107 vs 123 us), so one item never batches.
  bool split_batched(int s) {
    if (half_in || items[s].size() < 2 || items[s].size() > static_cast<std::size_t>(kMaxSplitJobs)) return false;
    double bytes_in = 0;
    for (const Item& it : items[s]) {
      if (it.landed) return false;
      bytes_in += static_cast<double>(it.pc->bytes());
    }
    if (bytes_in > static_cast<double>(env_int("DM_BATCH_SPLIT_MB", 64)) * (1 << 20)) return false;
    SplitJobs jobs;
    if (!make_jobs(s, &jobs)) return false;
    cuda_check(split_jobs(jobs, w.side), "split_jobs");
    w.stats.split_launches += 1;
    return true;
  }

  // Split jobs for the items of step s (false if a piece is not fusable).
  bool make_jobs(int s, SplitJobs* out) const {
    out->n = 0;
    std::int64_t t = 0;
    for (const Item& it : items[s]) {
      const Planes& pl = *it.pl;
      const std::int64_t off = plane_off(it);
      const SplitShape sh = split_shape(it);
      SplitJob& j = out->job[out->n++];
      j = SplitJob{};
      j.src = static_cast<const float*>(it.src);
      j.lds = it.lds;
      j.trans = sh.trans;
      j.rows = sh.rows;
      j.kcols = sh.cols;
      j.hi = pl.hi ? pl.hi + off : nullptr;
      j.lo = pl.lo ? pl.lo + off : nullptr;
      j.rmax = pl.rmax ? pl.rmax + it.pc->dst_row : nullptr;
      j.hi16 = pl.hi16 ? static_cast<char*>(pl.hi16) + off * 2 : nullptr;
      j.lo16 = pl.lo16 ? static_cast<char*>(pl.lo16) + off * 2 : nullptr;
      j.ldo = j.ldo16 = pl.ld;
      j.flag = it.landed ? flag : nullptr;
      j.flag_val = it.landed ? seq[s] : 0;
      j.t0 = t;
      if (!split_job_fusable(j)) return false;
      t += split_job_tiles(j);
    }
    out->t_begin = 0;
    out->t_end = t;
    return true;
  }

  // Split jobs of step s for the split warps of step s-1's GEMM launches.
  // Fused only when the carrying GEMM is long enough to hide the split: two
  // warps per SM split ~150 GB/s of input beside a ~300 TFLOP/s GEMM (a
  // narrow panel cannot hide a full panel's split -- that one runs as its own
  // full-machine kernels instead).
  bool fused_jobs(int s, SplitJobs* out) const {
    if (fuse_mode == 0 || items[s].empty() || items[s].size() > static_cast<std::size_t>(kMaxSplitJobs))
      return false;
    double bytes_in = 0, flops = 0;
    for (const Item& it : items[s]) bytes_in += static_cast<double>(it.pc->bytes());
    const std::int64_t kw = plan.k0[order[s - 1] + 1] - plan.k0[order[s - 1]];
    for (const Task& t : plan.tasks) {
      auto [mb, nb] = block_extent(S.table_.at(g.c).layout.grid, t.c);
      flops += 2.0 * mb * nb * static_cast<double>(kw);
    }
    // split-warp input rate and GEMM rate (DM_FUSE_SPLIT_GBS / DM_FUSE_GEMM_TFLOPS)
    const double split_bps = static_cast<double>(env_int("DM_FUSE_SPLIT_GBS", 150)) * 1e9;
    const double gemm_fps = static_cast<double>(env_int("DM_FUSE_GEMM_TFLOPS", f16x2() ? 450 : 300)) * 1e12;
    if (fuse_mode == 1 && bytes_in / split_bps > flops / gemm_fps) return false;
    if (f16x2()) {
      // the two-phase split (row maxima, grid handoff, split) must see all of a
      // plane row's tiles in one launch whose CTAs are all co-resident
      if (!exclusive || plan.tasks.size() != 1 || phase_ctr == nullptr) return false;
      out->phase_ctr = phase_ctr + s;
    }
    return make_jobs(s, out);
  }

  // The GEMM launches of step `step` (one per owned C block), carrying the
  // next panel's split tiles when `jobs` is set.
  void gemm_step(int step, SplitJobs* jobs) {
    const int p = order[step];
    const int buf = step % nbuf;
    if (split_ev[step]) cuda_check(cudaStreamWaitEvent(w.stream, split_ev[step], 0), "wait");
    const std::int64_t kw = plan.k0[p + 1] - plan.k0[p];
    cudaEvent_t tg = trace ? S.trace_event(w.stream) : nullptr;
    const double flops0 = w.stats.gemm_flops;
    const std::int64_t ntask = static_cast<std::int64_t>(plan.tasks.size());
    const std::int64_t split_tiles =
        jobs ? jobs->job[jobs->n - 1].t0 + split_job_tiles(jobs->job[jobs->n - 1]) : 0;
    for (std::int64_t ti = 0; ti < ntask; ++ti) {
      const Task& t = plan.tasks[ti];
      StoredBlock& cb = w.owned.at({g.c, t.c});
      const Planes& A = presplit ? spa[step][t.ra] : pa[t.ra][buf];
      const Planes& B = presplit ? spb[step][t.rb] : pb[t.rb][buf];
      Tf32x3Args a;
      a.mode = gemm_mode;
      a.a_mn = A.mn ? 1 : 0;
      a.b_mn = B.mn ? 1 : 0;
      a.a_hi = A.hi;
      a.a_lo = A.lo;
      a.a_hi16 = A.hi16;
      a.a_lo16 = A.lo16;
      a.lda = a.lda16 = A.ld;
      a.b_hi = B.hi;
      a.b_lo = B.lo;
      a.b_hi16 = B.hi16;
      a.b_lo16 = B.lo16;
      a.ldb = a.ldb16 = B.ld;
      a.c = cb.mem.f32();
      a.c_half = half_in ? 1 : 0;
      a.ldc = cb.cols;
      a.m = cb.rows;
      a.n = cb.cols;
      a.k = kw;
      a.alpha = static_cast<float>(g.alpha);
      // the first panel applies beta (beta == 0 never reads C, kernels.hpp:69-71);
      // later panels accumulate into what it wrote
      a.beta = step == 0 ? static_cast<float>(g.beta) : 1.0f;
      a.read_c = step == 0 ? (g.beta != 0.0 ? 1 : 0) : 1;
      a.cta_group = static_cast<int>(env_int("DM_CTA_GROUP", 0));
      a.flush_k = env_int("DM_FLUSH_K", 0);
      a.k_total = plan.k0.back();  // the chunk length follows the whole product's K
      a.group_m = static_cast<int>(env_int("DM_GROUP_M", 0));
      a.l2_policy = static_cast<int>(env_int("DM_L2_POLICY", 1));
      a.c_prefetch = static_cast<int>(env_int("DM_C_PREFETCH", -1));
      a.ksplit = static_cast<int>(env_int("DM_KSPLIT", 0));  // 0 auto, 1 off, >1 forced
      a.lockstep = lockstep;
      if (lockstep > 0) {
        const std::size_t need = tf32x3_sync_bytes(a);
        if (need > sync_bytes) {
          bufs.push_back(w.pool->acquire(need));
          sync = static_cast<unsigned*>(bufs.back().data());
          sync_bytes = bufs.back().capacity();
        }
        a.sync = sync;
        a.sync_bytes = sync_bytes;
      }
      if (jobs) {
        // the next panel's split tiles, spread evenly over this step's launches
        jobs->t_begin = split_tiles * ti / ntask;
        jobs->t_end = split_tiles * (ti + 1) / ntask;
        a.split = jobs;
        if (jobs->phase_ctr != nullptr) {  // kModeF16x2 (one launch): fresh maxima and handoff counter
          zero_rmax(step + 1, w.stream);
          cuda_check(cudaMemsetAsync(jobs->phase_ctr, 0, 4, w.stream), "memset phase counter");
        }
      }
      a.a_max = A.rmax;
      a.b_max = B.rmax;
      if (const std::size_t need = tf32x3_splitk_bytes(a)) {
        if (need > ksplit_ws_bytes) {
          bufs.push_back(w.pool->acquire(need));
          ksplit_ws = bufs.back().f32();
          ksplit_ws_bytes = bufs.back().capacity();
        }
        a.ws = ksplit_ws;
        a.ws_bytes = ksplit_ws_bytes;
      }
      S.record_timing(w, true);
      cuda_check(tf32x3_gemm(a, w.stream), "tf32x3_gemm");
      S.record_timing(w, false);
      w.stats.gemm_launches += 1;
      w.stats.gemm_flops += 2.0 * static_cast<double>(a.m) * a.n * a.k;
    }
    if (trace)
      w.trace.push_back({jobs ? "gemm+split" : "gemm", p, 0, w.stats.gemm_flops - flops0, tg,
                         S.trace_event(w.stream)});
    gemm_ev[step] = new_event();
    cuda_check(cudaEventRecord(gemm_ev[step], w.stream), "event");
  }

  // Double64: assemble op(A) rows / op(B) columns over the whole K, then the
  // bit-exact fp64 kernel (no split, no panels; gemm_f64.cu).
  void run_f64() {
    const std::int64_t K = plan.k0.back();
    const std::int64_t kp = std::max<std::int64_t>(1, K);
    auto assemble = [&](const std::vector<Range>& rs, std::vector<double*>& out) {
      for (const Range& r : rs) {
        bufs.push_back(w.pool->acquire(static_cast<std::size_t>(std::max<std::int64_t>(r.len, 1) * kp) * 8));
        double* panel = static_cast<double*>(bufs.back().data());
        out.push_back(panel);
        for (const Piece& pc : r.panels[0]) {
          bool remote = false;
          const double* src =
              static_cast<const double*>(S.source_ptr(w, pc.matrix, pc.coord, pol, &remote)) + pc.src_off;
          cuda_check(assemble_f64(src, pc.lds, pc.trans, pc.rows, pc.kcols, panel + pc.dst_row * kp + pc.dst_k, kp,
                                  w.side),
                     "assemble_f64");
          w.stats.split_launches += 1;
          (remote ? w.stats.peer_bytes_read : w.stats.local_bytes_read) += pc.bytes() * 2;
          if (remote) pulled_blocks[{pc.matrix, pc.coord}] += pc.bytes() * 2;
        }
      }
    };
    cudaEvent_t e = new_event();
    cuda_check(cudaEventRecord(e, w.stream), "event");
    cuda_check(cudaStreamWaitEvent(w.side, e, 0), "wait");
    std::vector<double*> pa64, pb64;
    if (K > 0) {
      assemble(plan.ar, pa64);
      assemble(plan.br, pb64);
    }
    cudaEvent_t done = new_event();
    cuda_check(cudaEventRecord(done, w.side), "event");
    cuda_check(cudaStreamWaitEvent(w.stream, done, 0), "wait");
    for (const Task& t : plan.tasks) {
      StoredBlock& cb = w.owned.at({g.c, t.c});
      S.record_timing(w, true);
      cuda_check(gemm_f64_exact(K > 0 ? pa64[t.ra] : nullptr, kp, K > 0 ? pb64[t.rb] : nullptr, kp,
                                static_cast<double*>(cb.mem.data()), cb.cols, cb.rows, cb.cols, K, g.alpha, g.beta,
                                g.beta != 0.0 ? 1 : 0, w.stream),
                 "gemm_f64_exact");
      S.record_timing(w, false);
      w.stats.gemm_launches += 1;
      w.stats.gemm_flops += 2.0 * static_cast<double>(cb.rows) * cb.cols * K;
    }
  }

  // one trace() record per foreign block this worker read in the command
  void log_pulls() {
    for (const auto& [key, bytes] : pulled_blocks)
      S.log_transfer(S.table_.at(key.matrix).layout.owner(key.coord), w.id, key.matrix, key.coord, bytes);
  }

  void run() {
    if (S.table_.at(g.a).precision == Precision::Double64) {
      run_f64();
      return log_pulls();
    }
    if (presplit) return run_presplit();
    setup();
    prepare(0);
    split_separate(0);
    commit_plane_cache();
    for (int step = 0; step < np; ++step) {
      SplitJobs jobs;
      bool fused_next = false;
      if (step + 1 < np) {
        prepare(step + 1);
        fused_next = fused_jobs(step + 1, &jobs);
        if (!fused_next) split_separate(step + 1);
      }
      gemm_step(step, fused_next ? &jobs : nullptr);
      if (fused_next) consumed_ev[step + 1] = gemm_ev[step];  // split inside this step's launches
    }
    log_pulls();
  }
};

void Session::drop_graphs(Worker& w, MatrixId id) {
  for (auto it = w.graphs.begin(); it != w.graphs.end();) {
    if (id == 0 || it->ids[0] == id || it->ids[1] == id || it->ids[2] == id) {
      cudaGraphExecDestroy(it->exec);
      it = w.graphs.erase(it);
    } else {
      ++it;
    }
  }
  if (id == 0) {
    w.plane_cache.clear();
  } else {
    for (auto it = w.plane_cache.begin(); it != w.plane_cache.end();)
      it = (!it->first.empty() && it->first[0] == static_cast<std::int64_t>(id)) ? w.plane_cache.erase(it) : ++it;
  }
}

namespace {
void add_stats(dm_worker_stats& a, const dm_worker_stats& d) {
  a.peer_bytes_read += d.peer_bytes_read;
  a.local_bytes_read += d.local_bytes_read;
  a.gemm_launches += d.gemm_launches;
  a.split_launches += d.split_launches;
  a.gemm_flops += d.gemm_flops;
}
dm_worker_stats sub_stats(const dm_worker_stats& a, const dm_worker_stats& b) {
  dm_worker_stats d{};
  d.peer_bytes_read = a.peer_bytes_read - b.peer_bytes_read;
  d.local_bytes_read = a.local_bytes_read - b.local_bytes_read;
  d.gemm_launches = a.gemm_launches - b.gemm_launches;
  d.split_launches = a.split_launches - b.split_launches;
  d.gemm_flops = a.gemm_flops - b.gemm_flops;
  return d;
}
}  // namespace

void Session::run_gemm(const GemmArgs& g, SourcePolicy pol) {
  struct Live {
    std::vector<DeviceBuffer> bufs;
    std::vector<cudaEvent_t> events;
  };
  std::vector<Live> live(P_);
  // Small single-panel commands are latency-bound: their per-worker launches
  // (splits, tensor-map encoding, GEMM, events) cost more host time than the
  // device spends on them.  A repeated command -- same operands, sources and
  // knobs -- replays the graph captured the first time instead (buffers kept
  // with the graph; a changed source pointer or plane-cache state is a new key).
  // Presplit (session_presplit.cpp): the owners split their A / B blocks
  // first -- after the asynchronous preamble, which then runs for every
  // worker here instead of in the loop below.
  const bool presplit = presplit_eligible(g, pol);
  if (!presplit && P_ > 1) {  // consumers read the operands' blocks on their owners' GPUs
    remote_read_.insert(g.a);
    remote_read_.insert(g.b);
  }
  if (presplit) {
    for (auto& wp : workers_) {
      if (!wp) continue;
      Worker& w = *wp;
      DeviceGuard guard(w.device);
      if (tracing() && !async_) w.trace_t0 = trace_event(w.stream);
      if (async_) {
        bound_inflight(w);
        wait_writes(w.side, g.a);
        wait_writes(w.side, g.b);
        wait_all(w.side, g.c);
        // the previous presplit command's plane reads, everywhere, end before
        // any owner overwrites its arena (this barrier orders them)
        for (auto& o : workers_)
          if (o && o->plane_reads) cuda_check(cudaStreamWaitEvent(w.side, o->plane_reads, 0), "wait plane readers");
        device_barrier(w.side, 1);
        wait_all(w.stream, g.c);
      } else {
        // operands were written by earlier commands on the compute stream
        if (!w.presplit_order)
          cuda_check(cudaEventCreateWithFlags(&w.presplit_order, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(w.presplit_order, w.stream), "event");
        cuda_check(cudaStreamWaitEvent(w.side, w.presplit_order, 0), "wait");
      }
    }
    HostScope hp("run_gemm: presplit owners");
    presplit_owners(g);
    // the compute stream covers the owner split even on a worker without C
    // blocks (a synchronous command ends by draining the compute streams)
    for (auto& wp : workers_)
      if (wp) {
        DeviceGuard guard(wp->device);
        cuda_check(cudaStreamWaitEvent(wp->stream, wp->presplit_done, 0), "wait presplit");
      }
  }
  const bool graphs_on = !async_ && !tracing() && !timing_ && !presplit && env_int("DM_GRAPHS", 1) != 0 &&
                         table_.at(g.a).precision != Precision::Double64;
  const double graph_max_flops = static_cast<double>(env_int("DM_GRAPH_MAX_GFLOP", 64)) * 1e9;
  const std::size_t graph_cap = static_cast<std::size_t>(std::max<std::int64_t>(1, env_int("DM_GRAPH_CACHE", 32)));
  for (auto& wp : workers_) {
    if (!wp) continue;
    Worker& w = *wp;
    DeviceGuard guard(w.device);
    WorkerPlan plan;
    {
      HostScope hp("run_gemm: plan_worker");
      plan = plan_worker(g, w.id, pol, presplit);
    }
    if (async_ && !presplit) {
      // pulls start once A and B are written everywhere; C is overwritten only
      // after its previous writes and reads (e.g. an async gather) finished
      bound_inflight(w);
      wait_writes(w.side, g.a);
      wait_writes(w.side, g.b);
      // C is about to be overwritten: every earlier local read of it (GEMMs
      // whose pulls / fused splits read it as an operand, async gathers)
      // finishes before this rank enters the barrier, so after the barrier no
      // rank still reads the old C while its owner's GEMM writes it.
      wait_all(w.side, g.c);
      device_barrier(w.side, 1);  // every rank, even one without C blocks
      wait_all(w.stream, g.c);
    }
    if (plan.tasks.empty()) continue;
    Live& lv = live[w.id];
    if (tracing() && !async_ && !presplit) w.trace_t0 = trace_event(w.stream);
    double work = 0;
    for (const Task& t : plan.tasks) {
      auto [mb, nb] = block_extent(table_.at(g.c).layout.grid, t.c);
      work += 2.0 * mb * nb * static_cast<double>(plan.k0.back());
    }
    const bool use_graph = graphs_on && plan.k0.size() == 2 && work <= graph_max_flops;
    GemmRun run(*this, w, g, pol, std::move(plan), lv.bufs, lv.events, presplit);
    if (!use_graph) {
      HostScope hr("run_gemm: GemmRun");
      run.run();
    } else {
      HostScope hr("run_gemm: graph");
      std::vector<std::uint64_t> sig;
      {
        HostScope hs("run_gemm: graph signature");
        sig = run.signature();
      }
      Worker::GraphEntry* hit = nullptr;
      for (auto& e : w.graphs)
        if (e.sig == sig) {
          hit = &e;
          break;
        }
      if (hit == nullptr) {
        HostScope hc("run_gemm: graph capture");
        // first time: capture the launches this command issues on the
        // worker's streams (the split stream joins through its events)
        const dm_worker_stats before = w.stats;
        cuda_check(cudaStreamBeginCapture(w.stream, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
        cudaGraph_t graph = nullptr;
        try {
          run.run();
        } catch (...) {
          cudaStreamEndCapture(w.stream, &graph);
          if (graph) cudaGraphDestroy(graph);
          throw;
        }
        cuda_check(cudaStreamEndCapture(w.stream, &graph), "cudaStreamEndCapture");
        Worker::GraphEntry e;
        const cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(ie, "cudaGraphInstantiate");
        e.sig = std::move(sig);
        e.delta = sub_stats(w.stats, before);
        e.pulls.assign(run.pulled_blocks.begin(), run.pulled_blocks.end());
        e.bufs = std::move(lv.bufs);
        lv.bufs.clear();
        e.ids[0] = g.a;
        e.ids[1] = g.b;
        e.ids[2] = g.c;
        if (w.graphs.size() >= graph_cap) {  // evict the least recently used
          auto lru = std::min_element(w.graphs.begin(), w.graphs.end(),
                                      [](const auto& x, const auto& y) { return x.last_use < y.last_use; });
          cudaGraphExecDestroy(lru->exec);
          w.graphs.erase(lru);
        }
        w.graphs.push_back(std::move(e));
        hit = &w.graphs.back();
        for (cudaEvent_t ev : lv.events) cudaEventDestroy(ev);
        lv.events.clear();
      } else {
        HostScope hc("run_gemm: graph replay");
        add_stats(w.stats, hit->delta);
        for (const auto& [key, bytes] : hit->pulls)
          log_transfer(table_.at(key.matrix).layout.owner(key.coord), w.id, key.matrix, key.coord, bytes);
        run.commit_plane_cache();
      }
      hit->last_use = ++w.graph_clock;
      HostScope hl("run_gemm: cudaGraphLaunch");
      cuda_check(cudaGraphLaunch(hit->exec, w.stream), "cudaGraphLaunch");
    }
    if (async_) {
      mark_write(w, w.stream, g.c);
      // A and B are read by the split stream and by the GEMMs' fused split warps
      for (cudaStream_t st : {w.side, w.stream}) {
        mark_read(w, st, g.a);
        mark_read(w, st, g.b);
      }
      // panel planes live until the last GEMM of this command has run
      Worker::Inflight f;
      cuda_check(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(f.done, w.stream), "event");
      f.bufs = std::move(lv.bufs);
      f.events = std::move(lv.events);
      f.events.push_back(f.done);
      w.inflight.push_back(std::move(f));
    }
  }
  if (async_) return;
  // Every split / pull of a command feeds the worker's GEMM stream (stream
  // waits, or the landing flag the GEMM's split warps spin on), so that
  // stream draining means the command's buffers are free; end_command()
  // synchronises the remaining streams.
  HostScope hsync("run_gemm: sync + release");
  for (auto& wp : workers_) {
    if (!wp) continue;
    DeviceGuard guard(wp->device);
    cuda_check(cudaStreamSynchronize(wp->stream), "gemm stream sync");
    for (cudaEvent_t e : live[wp->id].events) cudaEventDestroy(e);
    live[wp->id].bufs.clear();
  }
  streams_drained_ = true;
}

}  // namespace dm
