// flux_ring.cuh — the fused flux sweep of one direction as a warp-pipelined ring (product path).
//
// Same mathematics as flux_kernel (hgks_kernels.cuh): per face, the tangential reconstruction of the
// six face fields to the 2x2 Gauss points (A3: t1 pass, then t2 pass), the BGK flux of Eq. (6) with
// the time linearisation of Eq. (8) at each Gauss point (A4-A6) and the 4-point face quadrature (A7).
// What changes is the schedule:
//
//   * A block (one per SM, persistent) walks STRIPS of faces: TT1 = 8 faces along t1 at one normal
//     face index fn, L consecutive face rows along t2.  A face row (8 faces x 4 Gauss points) is one
//     warp's phase-C work unit.
//   * The t1 pass of face-field row l2 (the 12 lines of the tile at one t2) is computed ONCE per strip
//     into a ring of shared-memory rows; face row b reads rows b..b+4.  Along a strip of L rows the t1
//     pass costs (L+4)/L of the rows it serves instead of 12/8 for 8x8 tiles.
//   * No block-wide barriers.  Warp w handles face rows F = w, w+NW, ... of the block's row stream and
//     first PRODUCES ring row F+4 (and, at a strip start, row F for F < 4) from a per-warp staging
//     buffer filled by cp.async one production ahead, then CONSUMES rows F..F+4 (phase C).  Rows are
//     published with per-slot sequence numbers (release/acquire through __syncwarp + fence.cta) and
//     recycled with per-slot consumer counts, so warps synchronise only with the producers of the rows
//     they read: the t1 pass and the face-field copies of one warp overlap the Gauss-point flux of the
//     others.  Every producer wait points at strictly older face rows, so the pipeline cannot deadlock
//     (RING >= NW + 8 leaves one iteration of slack).
//   * A face row's five rows occupy consecutive slots: slots 0..3 are mirrored at RING..RING+3.
#pragma once
#include "hgks_kernels.cuh"

namespace hgks {

template <typename T>
struct RingCfg;
template <>
struct RingCfg<double> {
  static constexpr int NW = 16;    // warps per block (128 registers each: the whole register file)
  static constexpr int RING = 24;  // ring rows (+4 mirrored)
};
template <>
struct RingCfg<float> {
  static constexpr int NW = 24;  // 85 registers each
  static constexpr int RING = 32;
};

constexpr int RG_SP = TL1;             // staging: elements per (field, component) line row (12 lines)
constexpr int RG_ROW = 5 * SB_RC;      // elements of one ring row: [component][slot k][m][a] + pad
constexpr int RG_STAGE = 30 * RG_SP;   // elements of one warp's staging row (30 planes x 12 lines)

template <typename T>
constexpr size_t ring_smem_bytes() {
  return sizeof(T) * ((size_t)(RingCfg<T>::RING + 4) * RG_ROW + (size_t)RingCfg<T>::NW * RG_STAGE) +
         sizeof(int) * 2 * RingCfg<T>::RING;
}

// strip s of the sweep -> (t1 tile origin, t2 chunk origin, normal face index, strip length)
struct StripMap {
  int n1t, n2c, L, n2;
  __device__ __forceinline__ void decode(long long s, int& t10, int& t20, int& fn, int& Ls) const {
    const int i1 = (int)(s % n1t);
    const long long r = s / n1t;
    const int i2 = (int)(r % n2c);
    fn = (int)(r / n2c);
    t10 = i1 * TT1;
    t20 = i2 * L;
    Ls = min(L, n2 - t20);
  }
};

// face rows of a strip of length Ls that read ring row l2 (rows l2-4..l2)
__device__ __forceinline__ int row_consumers(int l2, int Ls) {
  const int lo = max(0, l2 - 4), hi = min(l2, Ls - 1);
  return max(0, hi - lo + 1);
}

// watchdog of the spin waits (~seconds): a schedule bug traps (the launch fails with an error) instead
// of hanging the device
constexpr unsigned RING_SPIN_LIMIT = 1u << 26;

__device__ __forceinline__ int ld_volatile(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void st_volatile(int* p, int v) { *(volatile int*)p = v; }

template <typename T, int DIR, int STAGE, bool PRF>
__global__ void __launch_bounds__(32 * RingCfg<T>::NW, 1)
    flux_ring_kernel(const T* __restrict__ ff, T* __restrict__ flux, Geo<T> g, GasK<T> gas, const Ctl* __restrict__ ctl,
                     StripMap sm, long long nstrips) {
  if (ctl->halt) return;
  constexpr int NW = RingCfg<T>::NW, RING = RingCfg<T>::RING;
  constexpr int A1 = (DIR + 1) % 3, A2 = (DIR + 2) % 3;  // tangent axes t1, t2 (O-23)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);                // [RING + 4][RG_ROW]
  T* stage_all = ring + (size_t)(RING + 4) * RG_ROW;       // [NW][RG_STAGE]
  int* seq = reinterpret_cast<int*>(stage_all + (size_t)NW * RG_STAGE);  // [RING] stream row + 1 held
  int* done = seq + RING;                                  // [RING] consumers done with that row
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T* stage = stage_all + (size_t)w * RG_STAGE;
  for (int k = threadIdx.x; k < 2 * RING; k += blockDim.x) seq[k] = 0;  // seq and done
  __syncthreads();  // the only block-wide barrier

  const int n1 = g.n[A1], n2 = g.n[A2];
  const FFLayout<T, DIR> FL = ff_layout<T, DIR>(g);
  const long long fstride = (long long)FL.nf * FL.nl;  // next (field, component) plane
  const long long G = gridDim.x;
  const long long my_strips = nstrips > blockIdx.x ? (nstrips - 1 - blockIdx.x) / G + 1 : 0;
  const long long nface_rows = my_strips * sm.L;
  const int L4 = sm.L + 4;  // stream rows per strip

  // ---- staging copy of face-field row l2 (t2 = t20 - 2 + l2) of strip j into this warp's buffer ----
  auto issue_stage = [&](long long j, int l2) {
    int t10, t20, fn, Ls;
    sm.decode(blockIdx.x + j * G, t10, t20, fn, Ls);
    const int t2 = min(t20 - 2 + l2, n2 + 1);
    const T* base = ff + (long long)fn * FL.nl;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(stage);
    constexpr int VEC = 16 / (int)sizeof(T);  // lines per 16-byte chunk
    constexpr int NCH = RG_SP / VEC;          // chunks per plane row
    if (t10 + TL1 - 2 <= n1 + 2) {            // whole tile row inside the array: 16-byte chunks
      for (int q = lane; q < 30 * NCH; q += 32) {
        const int pl = q / NCH, ch = q - pl * NCH;
        const T* src = base + pl * fstride + FL.line(t10 - 2 + ch * VEC, t2);
        const unsigned dst = sbase + (unsigned)((pl * RG_SP + ch * VEC) * (int)sizeof(T));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
    } else {  // ragged t1 edge: single lines, clamped
      for (int q = lane; q < 30 * RG_SP; q += 32) {
        const int pl = q / RG_SP, l1 = q - pl * RG_SP;
        const T* src = base + pl * fstride + FL.line(min(t10 + l1 - 2, n1 + 1), t2);
        const unsigned dst = sbase + (unsigned)((pl * RG_SP + l1) * (int)sizeof(T));
        if (sizeof(T) == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // first real ring row this warp produces for face row F (-1: none); the schedule (tests/ring_schedule.py
  // models it): face row bb produces the prologue rows l2 < 4 with l2 % L == bb, then row bb + 4
  auto first_prod = [&](long long F) -> int {
    if (F >= nface_rows) return -1;
    const long long j = F / sm.L;
    const int bb = (int)(F - j * sm.L);
    if (bb < 4) return bb;
    int t10, t20, fn, Ls;
    sm.decode(blockIdx.x + j * G, t10, t20, fn, Ls);
    return bb < Ls ? bb + 4 : -1;
  };

  // ---- t1 pass (A3) of the staged row into ring slot(s): items (a, m, c), 80 per row ----------------
  // Every stream row is produced exactly once, by the warp of face row l2 - 4 (rows 0..3: face row
  // l2 % L).  Rows past a ragged strip end (l2 >= Ls + 4) get a NULL production (real = false): no data,
  // but the slot hand-over (wait for the previous occupant's consumers) still happens, so every slot
  // transition is guarded.
  auto produce = [&](long long j, int l2, bool real) {
    const long long R = j * L4 + l2;
    const int sl = (int)(R % RING);
    if (R >= RING) {  // recycle: every consumer of the row R - RING must be done with it
      const long long Rp = R - RING;
      const long long jp = Rp / L4;
      const int l2p = (int)(Rp - jp * L4);
      int t10p, t20p, fnp, Lsp;
      sm.decode(blockIdx.x + jp * G, t10p, t20p, fnp, Lsp);
      const int need = row_consumers(l2p, Lsp);
      // the slot must hold the previous occupant (its producer has run: producers of one slot then run
      // in stream order, whatever the warps' drift) and every consumer of it must be done
      if (lane == 0) {
        unsigned spins = 0;
        while (ld_volatile(&seq[sl]) != (int)(Rp + 1) || ld_volatile(&done[sl]) < need) {
          __nanosleep(32);
          if (++spins > RING_SPIN_LIMIT) __trap();  // schedule bug: fail the launch instead of hanging
        }
        st_volatile(&done[sl], 0);
      }
      __syncwarp();
    }
    if (!real) {
      if (lane == 0) st_volatile(&seq[sl], (int)(R + 1));
      return;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();  // the staged row landed for every lane
    for (int item = lane; item < 80; item += 32) {
      const int a = item & 7, m = (item >> 3) & 1, c = item >> 4;
      T wv[5], wd[5];
#pragma unroll
      for (int r = 0; r < 5; ++r) {  // m = 1: mirrored weights wv[1][r] = wv[0][4-r], wd[1][r] = -wd[0][4-r]
        wv[r] = m ? T(kWV0(4 - r)) : T(kWV0(r));
        wd[r] = m ? -T(kWD0(4 - r)) : T(kWD0(r));
      }
      T o[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) o[k] = T(0);
      const T* src = stage + c * RG_SP + a;
#pragma unroll
      for (int r = 0; r < 5; ++r) {
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          const T x = src[f * 5 * RG_SP + r];
          o[f] += wv[r] * x;
          if (f == 0) o[6] += wd[r] * x;
          if (f == 1) o[7] += wd[r] * x;
          if (f == 4) o[8] += wd[r] * x;
        }
      }
      T* dst = ring + (size_t)sl * RG_ROW + c * SB_RC + m * TT1 + a;
#pragma unroll
      for (int k = 0; k < NB; ++k) dst[k * SB_K] = o[k];
      if (sl < 4) {
        T* dm = dst + (size_t)RING * RG_ROW;
#pragma unroll
        for (int k = 0; k < NB; ++k) dm[k * SB_K] = o[k];
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      st_volatile(&seq[sl], (int)(R + 1));
    }
  };

  const T dt = T(ctl->dt);
  const int a = lane & 7, m = (lane >> 3) & 1, nn = lane >> 4;
  const T sgn = nn ? T(-1) : T(1);
#ifndef HGKS_ROW_MIRROR64
#define HGKS_ROW_MIRROR64 1
#endif
  constexpr bool kRowMirror = sizeof(T) == 8 && HGKS_ROW_MIRROR64;
  T wvl[5], wdl[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    wvl[r] = (!kRowMirror && nn) ? T(kWV0(4 - r)) : T(kWV0(r));
    wdl[r] = (!kRowMirror && nn) ? -T(kWD0(4 - r)) : T(kWD0(r));
  }

  {  // prefetch this warp's first production
    const int p = first_prod(w);
    if (p >= 0) issue_stage(0, p);
  }
  for (long long F = w; F < nface_rows; F += NW) {
    const long long j = F / sm.L;
    const int bb = (int)(F - j * sm.L);
    int t10, t20, fn, Ls;
    sm.decode(blockIdx.x + j * G, t10, t20, fn, Ls);
    // ---- produce: the strip's prologue rows l2 < 4 with l2 % L == bb, then row bb + 4 ------------
    bool staged = true;  // the prefetch holds this face row's first real production
    for (int l2 = bb; l2 < 4; l2 += sm.L) {
      if (!staged) issue_stage(j, l2);
      produce(j, l2, true);
      staged = false;
    }
    if (bb < Ls && !staged) issue_stage(j, bb + 4);
    produce(j, bb + 4, bb < Ls);
    {  // prefetch the next production of this warp (its staging buffer is free again)
      const int p = first_prod(F + NW);
      if (p >= 0) issue_stage((F + NW) / sm.L, p);
    }
    if (bb >= Ls) continue;  // face row beyond a ragged strip end
    // ---- consume: wait for rows bb..bb+4 --------------------------------------------------------
    const long long R0 = j * L4 + bb;
    if (lane < 5) {
      const int sl = (int)((R0 + lane) % RING);
      unsigned spins = 0;
      while (ld_volatile(&seq[sl]) != (int)(R0 + lane + 1)) {
        __nanosleep(20);
        if (++spins > RING_SPIN_LIMIT) __trap();
      }
      __threadfence_block();
    }
    __syncwarp();
    const int slot0 = (int)(R0 % RING);
    // ---- phase C: one thread per Gauss point (as flux_kernel) ------------------------------------
    const int t2f = t20 + bb;  // this face row's t2 index
    const T ih1 = g.jg[A1][m * n1 + min(t10 + a, n1 - 1)], ih2 = g.jg[A2][nn * n2 + min(t2f, n2 - 1)];
    const T* row0 = ring + (size_t)slot0 * RG_ROW + m * TT1 + a + (kRowMirror && nn ? 4 : 0) * RG_ROW;
    const int rstep = (kRowMirror && nn) ? -RG_ROW : RG_ROW;
    auto tv = [&](int c, int k) {
      asm volatile("" ::: "memory");
      T v = T(0);
#pragma unroll
      for (int r = 0; r < 5; ++r) v += (kRowMirror ? wv0<T>(r) : wvl[r]) * row0[r * rstep + c * SB_RC + k * SB_K];
      return v;
    };
    auto td = [&](int c, int k) {
      asm volatile("" ::: "memory");
      T v = T(0);
#pragma unroll
      for (int r = 0; r < 5; ++r) v += (kRowMirror ? wd0<T>(r) : wdl[r]) * row0[r * rstep + c * SB_RC + k * SB_K];
      return kRowMirror ? sgn * v : v;
    };
    auto tvd = [&](int c, int k, T& v, T& d) {
      asm volatile("" ::: "memory");
      v = T(0);
      d = T(0);
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const T x = row0[r * rstep + c * SB_RC + k * SB_K];
        v += (kRowMirror ? wv0<T>(r) : wvl[r]) * x;
        d += (kRowMirror ? wd0<T>(r) : wdl[r]) * x;
      }
      if (kRowMirror) d *= sgn;
    };
    GpFlux<T, STAGE == 1, PRF> gf;
    T d2l[5], d2r[5];
    {
      T Wl[5], Wr[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        tvd(c, 0, Wl[c], d2l[c]);
        tvd(c, 1, Wr[c], d2r[c]);
      }
      gf.begin(gas, Wl, Wr, dt, T(1) / dt);
    }
    gf.template add_side<+1>([&](int i, T (&d)[5]) {
#pragma unroll
      for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 2) : (i == 1 ? tv(c, 6) * ih1 : d2l[c] * ih2);
    });
    gf.template add_side<-1>([&](int i, T (&d)[5]) {
#pragma unroll
      for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 3) : (i == 1 ? tv(c, 7) * ih1 : d2r[c] * ih2);
    });
    gf.add_equilibrium([&](int i, T (&d)[5]) {
#pragma unroll
      for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 5) : (i == 1 ? tv(c, 8) * ih1 : td(c, 4) * ih2);
    });
    // every ring read of this face row is done (its values fed the flux): release the five rows
    __syncwarp();
    if (lane < 5) {
      __threadfence_block();
      atomicAdd(&done[(int)((R0 + lane) % RING)], 1);
    }
    T F5[5], dF5[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      F5[k] = gf.F[k];
      dF5[k] = gf.dF[k];
    }
    // 2x2 Gauss quadrature, omega_mn = 1/4 (O-8): the face's Gauss points sit at lanes a, a+8, a+16, a+24
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (STAGE == 1) {
        F5[k] += __shfl_xor_sync(0xffffffffu, F5[k], 8);
        F5[k] += __shfl_xor_sync(0xffffffffu, F5[k], 16);
      }
      dF5[k] += __shfl_xor_sync(0xffffffffu, dF5[k], 8);
      dF5[k] += __shfl_xor_sync(0xffffffffu, dF5[k], 16);
    }
    const int f1 = t10 + a, f2 = t2f;
    if (lane < 8 && f1 < n1 && f2 < n2) {
      int cd[3];
      cd[DIR] = fn;
      cd[A1] = f1;
      cd[A2] = f2;
      const int fx = g.n[0] + (DIR == 0), fy = g.n[1] + (DIR == 1), fz = g.n[2] + (DIR == 2);
      const long long nface = (long long)fx * fy * fz;
      const long long id = ((long long)cd[2] * fy + cd[1]) * fx + cd[0];
      const int gc[5] = {0, 1 + DIR, 1 + A1, 1 + A2, 4};
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        if (STAGE == 1) flux[gc[k] * nface + id] = T(0.25) * F5[k];
        flux[(5 + gc[k]) * nface + id] = T(0.25) * dF5[k];
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace hgks
