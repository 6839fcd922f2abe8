// hadacore.cu -- C ABI (include/hadacore.h) of the B200-native batched normalized
// Walsh-Hadamard transform: argument validation, per-(n, dtype) kernel dispatch,
// launch configuration, and the pipelined host-buffer entry point.
// "P:NN" = /root/reference/PAPER.md line NN.
#include <cuda_runtime.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>

#include <type_traits>

#include "../../include/hadacore.h"
#include "fwht_kernel.cuh"
#include "fwht_small.cuh"
#include "fwht_f32.cuh"
#include "quant_lab.cuh"
#include "fwht_quant_tc.cuh"

namespace hadacore {
namespace {

constexpr int kVersion = 100;  // 0.1.0
constexpr int kMaxDevices = 64;

std::atomic<int> g_sm_count[kMaxDevices];

int sm_count(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return 148;
  int v = g_sm_count[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    g_sm_count[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Per-n launch configuration.  A CTA = NT compute
// warps + 1 producer warp, a STAGES-deep ring of tiles of ~TILE_KB KiB (whole rows;
// one row per tile for n = 2^14, 2^15), rows split into teams of P warps (n > 256)
// that synchronise with named barriers; the grid has one CTA per tile and CTAs steal
// tiles through cluster launch control.  The HC_* macros let tools/*.sh build A/B
// variants; the defaults are the tuned values.
// Tuned per n on B200 in bench.py's launch sequence under CLC scheduling (paired
// sweeps, profiles/r01_tune_sweep16_clc_retune.txt): compute warps, tile KiB, ring
// stages, work items per warp in flight, CTAs per SM.
template <int N> struct Tuned0;
template <> struct Tuned0<128>   { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<256>   { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<512>   { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<1024>  { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<2048>  { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<4096>  { static constexpr int nt = 16, tkb = 16, st = 4, u = 1, ctas = 1; };
template <> struct Tuned0<8192>  { static constexpr int nt = 16, tkb = 16, st = 6, u = 1, ctas = 1; };
template <> struct Tuned0<16384> { static constexpr int nt = 16, tkb = 32, st = 4, u = 1, ctas = 1; };  // r01_ab_transform_tune.txt
template <> struct Tuned0<32768> { static constexpr int nt = 16, tkb = 64, st = 3, u = 1, ctas = 1; };

#ifdef HC_TTUNE  // A/B builds: override the transform's table for n = HC_TTUNE_N
struct TMacro { static constexpr int nt = HC_TNT, tkb = HC_TTKB, st = HC_TST, u = 1, ctas = HC_TCTAS; };
template <int N> struct Tuned : std::conditional_t<(N == HC_TTUNE_N), TMacro, Tuned0<N>> {};
#else
template <int N> struct Tuned : Tuned0<N> {};
#endif

// Fused quantization (QT >= 0): its epilogue (row max, team barrier, code pass) makes
// a tile's critical path longer, so more independent pipelines per SM win: 3 CTAs of
// 8 consumer warps with 32 KiB tiles in a 2-stage ring (paired sweeps,
// profiles/r01_quant_sweep*.txt: +20-60 % over the transform's table at n = 2^10..2^14).
// n >= 512 keeps each warp's phase-B results (IW = tile / (nt * 512 B) chunks of 8 fp32
// per lane) in registers across the row-max barrier, so tiles are sized to IW = 4..8
// and the CTA count to the register file (paired sweeps, profiles/r01_quant_tune_v3.txt).  HC_QTUNE = "nt,tkb,st,ctas"
// overrides n = 512..8192 (A/B builds).
// round 2: 4 items in flight per warp (u = 4; E4M3/INT8 n = 512..8192 sweep 6.17 -> 6.48 TB/s), 4 warps x 4 CTAs
// at n = 2048 and 8192 (+2..5 % there; profiles/r02_quant_u_ab.txt)
template <int N> struct TunedQ0     { static constexpr int nt = 8, tkb = 16, st = 3, u = 4, ctas = 3; };
template <> struct TunedQ0<2048>    { static constexpr int nt = 4, tkb = 16, st = 3, u = 4, ctas = 4; };
template <> struct TunedQ0<128>     { static constexpr int nt = 8, tkb = 32, st = 2, u = 4, ctas = 3; };  // u = 4 (was 1): INT4 +16 %, Q/K quant (profiles/r02_quant_n128_ab.txt)
template <> struct TunedQ0<256>     { static constexpr int nt = 8, tkb = 32, st = 2, u = 2, ctas = 3; };  // u = 2 (was 1): INT4 +2..5 %
template <> struct TunedQ0<8192>    { static constexpr int nt = 4, tkb = 16, st = 3, u = 4, ctas = 4; };
template <> struct TunedQ0<16384>   { static constexpr int nt = 8, tkb = 32, st = 3, u = 1, ctas = 2; };
template <> struct TunedQ0<32768>   { static constexpr int nt = 16, tkb = 64, st = 3, u = 1, ctas = 1; };
#ifdef HC_QTUNE  // A/B builds: HC_QTUNE_N = the n to override (0: every n in 512..8192)
#ifndef HC_QU
#define HC_QU 1
#endif
struct QMacro { static constexpr int nt = HC_QNT, tkb = HC_QTKB, st = HC_QST, u = HC_QU, ctas = HC_QCTAS; };
template <int N>
struct TunedQ : std::conditional_t<(HC_QTUNE_N == N || (HC_QTUNE_N == 0 && N >= 512 && N <= 8192)), QMacro,
                                   TunedQ0<N>> {};
#else
template <int N> struct TunedQ : TunedQ0<N> {};
#endif

// Rows shorter than 128 (NEXT-2, fwht_small_kernel): 8 consumer warps, 32 KiB tiles,
// 4-stage ring; U items per lane in flight (an item is 8 elements for n <= 8, a row
// of n elements otherwise).
template <int N> struct TunedS {
  static constexpr int nt = 8, tkb = 32, st = 4, u = N <= 8 ? 4 : (N == 16 ? 2 : 1);
};
// The same kernel with the fused quantization epilogue (codes straight from registers):
// one item per lane in flight (U = 1) and, for n <= 8, 16 consumer warps (paired sweep,
// profiles/r01_ab_small_quant.txt: n = 2..32 from 3.1-5.7 to 5.6-6.6 TB/s).
// HC_SQTUNE = "n: nt,tkb,st,u" overrides it (A/B builds, tools/ab_small_quant.sh; n = 0: every n).
template <int N> struct TunedSQ0 { static constexpr int nt = 8, tkb = 32, st = 4, u = 1; };
template <> struct TunedSQ0<2> { static constexpr int nt = 16, tkb = 16, st = 4, u = 1; };
template <> struct TunedSQ0<4> { static constexpr int nt = 16, tkb = 16, st = 4, u = 1; };
template <> struct TunedSQ0<8> { static constexpr int nt = 16, tkb = 32, st = 4, u = 1; };
template <> struct TunedSQ0<16> { static constexpr int nt = 8, tkb = 16, st = 4, u = 1; };
template <> struct TunedSQ0<32> { static constexpr int nt = 8, tkb = 16, st = 4, u = 1; };
#ifdef HC_SQTUNE
struct SQMacro { static constexpr int nt = HC_SQNT, tkb = HC_SQTKB, st = HC_SQST, u = HC_SQU; };
template <int N> struct TunedSQ : std::conditional_t<(HC_SQTUNE_N == N || HC_SQTUNE_N == 0), SQMacro, TunedSQ0<N>> {};
#else
template <int N> struct TunedSQ : TunedSQ0<N> {};
#endif

// Small problems (n <= 256, contiguous, <= 4 MiB: e.g. BASELINE C1, 1024 x 256 fp16):
// launch-latency-bound, so tiles of 2 KiB spread the work over more SMs and shorten each
// CTA's load -> compute -> store chain (C1: 1.93 -> 1.71 us per launch in a CUDA graph,
// profiles/r01_ab_c1.txt).  Selected at run time as the QT_SMALLM instantiation.
struct TunedSmallM { static constexpr int nt = 4, tkb = 2, st = 2, u = 1, ctas = 1; };
constexpr int QT_SMALLM = -2;  // kernels treat every QT < 0 as the plain transform

// Mid-size problems (n = 512..4096, contiguous, at most HC_MIDM_MB MiB of input, i.e. up to
// 2^26 elements -- BASELINE C4 is 2^26): the whole launch is a few tiles per SM, so the ramp
// (first loads) and the tail (last tiles' phase 1 -> phase 2 -> store chain) dominate; 8 KiB
// tiles and 2 CTAs of 8 consumer warps per SM start more independent pipelines.  Selected at
// run time as the QT_MIDM instantiation.  Paired sweep (tools/midsize.py, 8 variants x n x
// 2^22..2^26, profiles/r02_midsize.md): n = 4096 at 2^24 elements 6243 -> 6494 GB/s warm
// (n = 256: 6772); n = 8192..32768 were no better and keep the main table.  HC_MIDM_* macros
// override the table for A/B builds (HC_MIDM_MB=0 disables it).
#ifndef HC_MIDM_MB
#define HC_MIDM_MB 128
#endif
#ifndef HC_MIDM_MAXN
#define HC_MIDM_MAXN 4096
#endif
template <int N> struct TunedMidM0 { static constexpr int nt = 8, tkb = 8, st = 4, u = 1, ctas = 2; };
#ifdef HC_MIDM_NT
template <int N> struct TunedMidM {
#ifndef HC_MIDM_U
#define HC_MIDM_U 1
#endif
  static constexpr int nt = HC_MIDM_NT, tkb = HC_MIDM_TKB, st = HC_MIDM_ST, u = HC_MIDM_U, ctas = HC_MIDM_CTAS;
};
#else
template <int N> struct TunedMidM : TunedMidM0<N> {};
#endif
constexpr int QT_MIDM = -3;

#ifdef HC_TUNE  // tools/tune.py: one configuration for every n, from -D macros
template <int N, int QT>
struct Knobs { static constexpr int nt = HC_NT, tkb = HC_TILE_KB, st = HC_STAGES, u = HC_U, ctas = HC_CTAS; };
#else
template <int N, int QT>
struct Knobs
    : std::conditional_t<(QT >= 0), TunedQ<N>,
                         std::conditional_t<(QT == QT_SMALLM), TunedSmallM,
                                            std::conditional_t<(QT == QT_MIDM), TunedMidM<N>, Tuned<N>>>> {};
#endif

template <int N, int QT = -1>
struct Cfg {
  using K = Knobs<N, QT>;
  static constexpr int nt = K::nt;
  static constexpr int rows = (K::tkb * 1024) / (2 * N) > 0 ? (K::tkb * 1024) / (2 * N) : 1;
  static constexpr int tile_bytes = rows * 2 * N;
  // more CTAs per SM only if each can still hold a double-buffered ring
  static constexpr int ctas = ((227 * 1024 / K::ctas - 256) / tile_bytes) >= 2 ? K::ctas : 1;
  static constexpr int max_stages = (227 * 1024 / ctas - 1408) / tile_bytes;
  static constexpr int stages = K::st < max_stages ? K::st : max_stages;
  static constexpr int nteams = N <= 256 ? 1 : (rows < nt ? rows : nt);
  static constexpr int p = N <= 256 ? 1 : nt / nteams;
  static constexpr int u = K::u;
  static_assert(stages >= 2, "need at least a double-buffered ring");
};

// cuTensorMapEncodeTiled from the driver, fetched through the runtime (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Row layout of one call: rows (i, j), i < m_outer, j < m_inner,
// at base + i*so + j*si elements; contiguous m x n is {m, 1, n, n}.
struct Layout {
  int64_t m_outer, m_inner;
  int64_t in_so, in_si, out_so, out_si;
};

// Tile shape for TILE_ROWS rows: bi (power of two) inner x bo outer rows.
RowGrid make_grid(const Layout& L, int tile_rows) {
  int bi = 1;
  while (bi * 2 <= tile_rows && bi * 2 <= L.m_inner) bi *= 2;
  int lbi = 0;
  while ((1 << lbi) < bi) ++lbi;
  RowGrid g{};
  g.m_outer = L.m_outer;
  g.m_inner = L.m_inner;
  g.out_so = L.out_so;
  g.out_si = L.out_si;
  g.lbi = lbi;
  g.bo = tile_rows / bi;
  g.nib = (L.m_inner + bi - 1) / bi;
  g.num_tiles = ((L.m_outer + g.bo - 1) / g.bo) * g.nib;
  return g;
}

// 3-D view (n elements, inner row, outer row) for fwht_kernel (n <= 256), box (n, bi, bo).
bool encode_small_map(CUtensorMap* map, const void* base, const Layout& L, int64_t so, int64_t si, int n,
                      const RowGrid& g) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(n), cuuint64_t(L.m_inner), cuuint64_t(L.m_outer)};
  cuuint64_t strides[2] = {cuuint64_t(2) * cuuint64_t(si), cuuint64_t(2) * cuuint64_t(so)};
  cuuint32_t box[3] = {cuuint32_t(n), cuuint32_t(1u << g.lbi), cuuint32_t(g.bo)};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 5-D view for fwht_rows_kernel (n >= 512): (64 elements, chunk c of 256 elements
// [stride 512 B], 128-byte segment s of the chunk [stride 128 B], inner row, outer
// row); box (64, C, 4, bi, bo) with SWIZZLE_128B,
// or (64, C, 1, 1, 1) per (row, segment) in SEG mode.
bool encode_rows_map(CUtensorMap* map, const void* base, const Layout& L, int64_t so, int64_t si, int n,
                     const RowGrid& g, bool seg) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const int C = n / 256;
  cuuint64_t dims[5] = {64, cuuint64_t(C), 4, cuuint64_t(L.m_inner), cuuint64_t(L.m_outer)};
  cuuint64_t strides[4] = {512, 128, cuuint64_t(2) * cuuint64_t(si), cuuint64_t(2) * cuuint64_t(so)};
  cuuint32_t box[5] = {64, cuuint32_t(C), seg ? 1u : 4u, seg ? 1u : cuuint32_t(1u << g.lbi), seg ? 1u : cuuint32_t(g.bo)};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Launch with programmatic dependent launch (PDL): the grid may be scheduled while
// the previous kernel on the stream drains, runs its prologue (barrier init, TMA
// descriptor prefetch, constants) and waits in griddepcontrol.wait before its first
// global-memory access -- so it is safe whatever the previous kernel wrote or read.
#ifndef HC_NO_PDL
constexpr bool kPdl = true;
#else
constexpr bool kPdl = false;
#endif
template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kern, int grid, int block, int smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = kPdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern>
bool ensure_smem_attr(Kern kern, int smem, std::atomic<uint64_t>& done, int dev) {
  const uint64_t bit = (dev >= 0 && dev < 64) ? (1ull << dev) : 0;
  if (bit && (done.load(std::memory_order_relaxed) & bit)) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return false;
  done.fetch_or(bit, std::memory_order_relaxed);
  return true;
}

// Fused quantization on tcgen05 + TMEM (fwht_quant_tc.cuh) for rows of n >= HC_QTC_MINN
// (contiguous or row grids): NA phase-A warps, NE epilogue warps, ST 64 KiB stages
// (DESIGN.md §5).
// HC_QTC_MINN = 0 disables it (A/B builds: the fwht_rows_kernel epilogue for every n).
#ifndef HC_QTC_MINN
#define HC_QTC_MINN 16384  // E4M3 / INT8; per-(qtype, n) A/B: profiles/r02_quant_tc_ab.txt
#endif
#ifndef HC_QTC_MINN4
#define HC_QTC_MINN4 16384  // INT4 from this n, plus n = HC_QTC_INT4_N below (after the register epilogue's u = 4
                           // retune it leads at n = 1024..8192 by 1..10 %, the tcgen05 kernel at 512 by 6..11 %:
                           // profiles/r02_quant_u_ab.txt; before it, tcgen05 led from 512: r02_quant_tc_small_c_ab.txt)
#endif
#ifndef HC_QTC_INT4_N
#define HC_QTC_INT4_N 512
#endif
#ifndef HC_QTC_NA
#define HC_QTC_NA 8
#endif
#ifndef HC_QTC_NE
#define HC_QTC_NE 4
#endif
#ifndef HC_QTC_ST
#define HC_QTC_ST 3  // stages when the codes are staged in them (HC_QTC_CB = 0)
#endif
#ifndef HC_QTC_ST_CB
#define HC_QTC_ST_CB 2  // stages with separate code buffers (HC_QTC_CB = 1, the default)
#endif
#ifndef HC_QTC_EG
#define HC_QTC_EG 2  // epilogue groups on alternate tiles (INT4 +4.5 %: profiles/r02_quant_tc_eg.txt)
#endif

// 5-D view (64 elements, chunk [512 B], inner row, outer row, 64-element segment [128 B])
// of a row grid; box (64, C, bi, bo, 2) with bi * bo = 128 / C rows, SWIZZLE_128B: half a
// segment-major tile of 128 chunk lines per segment (fwht_quant_tc_kernel loads two).
bool encode_tc_map(CUtensorMap* map, const void* base, const Layout& L, int n, const RowGrid& g) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const int C = n / 256;
  cuuint64_t dims[5] = {64, cuuint64_t(C), cuuint64_t(L.m_inner), cuuint64_t(L.m_outer), 4};
  cuuint64_t strides[4] = {512, cuuint64_t(2) * cuuint64_t(L.in_si), cuuint64_t(2) * cuuint64_t(L.in_so), 128};
  cuuint32_t box[5] = {64, cuuint32_t(C), cuuint32_t(1u << g.lbi), cuuint32_t(g.bo), 2};  // half a tile
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D view (128 bytes, 128-byte line of a row's codes, inner row, outer row) of the codes
// out_q (contiguous rows in (i, j) order); box (128, lines per row, bi, bo), SWIZZLE_128B:
// fwht_quant_tc_kernel stages a tile's codes swizzled and stores them with one TMA copy.
bool encode_tc_qmap(CUtensorMap* map, void* q, const Layout& L, int code_bytes, const RowGrid& g) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return false;
  const int lines = code_bytes / 128;
  cuuint64_t dims[4] = {128, cuuint64_t(lines), cuuint64_t(L.m_inner), cuuint64_t(L.m_outer)};
  cuuint64_t strides[3] = {128, cuuint64_t(code_bytes), cuuint64_t(code_bytes) * cuuint64_t(L.m_inner)};
  cuuint32_t box[4] = {128, cuuint32_t(lines), cuuint32_t(1u << g.lbi), cuuint32_t(g.bo)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, q, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N, int DT, int QT>
hadacore_status_t launch_qtc(const void* in, uint8_t* out_q, float* row_scale, const Layout& L, float scale,
                             cudaStream_t stream) {
  constexpr int NA = HC_QTC_NA, NE = HC_QTC_NE, EG = HC_QTC_EG;
  constexpr int ST = kTcCodeBuf ? (tc_h64<QT>() ? 3 : HC_QTC_ST_CB) : HC_QTC_ST;  // H64 frees room for a third stage
  constexpr int smem = tc_smem_bytes<ST, NE, QT, EG>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  auto kern = fwht_quant_tc_kernel<N, DT, QT, ST, NA, NE, EG>;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  const RowGrid g = make_grid(L, 128 / (N / 256));
  const int64_t max_ctas = kClc ? int64_t(INT32_MAX) : int64_t(sm_count(dev));
  const int grid = int(g.num_tiles < max_ctas ? g.num_tiles : max_ctas);
  CUtensorMap tin, tq;
  if (!encode_tc_map(&tin, in, L, N, g) || !encode_tc_qmap(&tq, out_q, L, QT == QT_INT4 ? N / 2 : N, g))
    return HADACORE_ERR_CUDA;
  // phase A's constants carry 2^-stage_shift(mask_a); H_128 is +-1
  const float s_res = std::ldexp(scale, stage_shift(PlanL<log2_n<N>() - 8>::mask_a));
  if (launch_pdl(kern, grid, (EG * NE + NA + 2) * 32, smem, stream, tin, tq, row_scale, g, s_res) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

template <int N, int DT, int QT>
hadacore_status_t launch(const void* in, void* out, uint8_t* out_q, float* row_scale, const Layout& L, float scale,
                         cudaStream_t stream) {
  if constexpr (QT >= 0 && N >= 512 && HC_QTC_MINN > 0 &&
                (N >= (QT == QT_INT4 ? HC_QTC_MINN4 : HC_QTC_MINN) || (QT == QT_INT4 && N == HC_QTC_INT4_N))) {
    return launch_qtc<N, DT, QT>(in, out_q, row_scale, L, scale, stream);
  }
#ifndef HC_TUNE
  if constexpr (N <= 256 && QT == QT_NONE) {
    if (L.m_inner == 1 && L.in_so == N && L.out_so == N && L.m_outer * N * 2 <= (int64_t(4) << 20))
      return launch<N, DT, QT_SMALLM>(in, out, out_q, row_scale, L, scale, stream);
  }
  if constexpr (N > 256 && N <= HC_MIDM_MAXN && QT == QT_NONE && HC_MIDM_MB > 0) {
    if (L.m_inner == 1 && L.in_so == N && L.out_so == N && L.m_outer * N * 2 <= (int64_t(HC_MIDM_MB) << 20))
      return launch<N, DT, QT_MIDM>(in, out, out_q, row_scale, L, scale, stream);
  }
#endif
  using C = Cfg<N, QT>;
  constexpr bool seg = seg_mode(N, C::rows);
  // + full[], done[][<=16] and the fused-quantization row-max scratch (one float per warp)
  constexpr int smem = C::stages * C::tile_bytes + int(sizeof(SchedCtl)) + 17 * C::stages * 8 +
                       4 * C::nt * (N > 256 ? C::rows : 1);
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  const RowGrid g = make_grid(L, C::rows);
  // CLC scheduling (default): one CTA per tile, resident CTAs steal the rest;
  // HC_STATIC_SCHED: persistent grid of one CTA per SM with round-robin tiles
  const int64_t max_ctas = kClc ? int64_t(INT32_MAX) : int64_t(sm_count(dev)) * C::ctas;
  const int grid = int(g.num_tiles < max_ctas ? g.num_tiles : max_ctas);
  // the per-stage constants multiply by exact powers of two 2^-E; fold the rest of
  // `scale` into the fp32 epilogue of the last stage.
  const float s_res = std::ldexp(scale, total_shift<N>());
  if constexpr (N <= 256) {
    // contiguous m x n in and out: 1-D bulk loads and flat epilogue addressing
    const bool flat = L.m_inner == 1 && L.in_so == N && (QT >= 0 || L.out_so == N);
    auto kern = flat ? fwht_kernel<N, DT, C::rows, C::stages, C::nt, C::p, C::u, C::ctas, QT, true>
                     : fwht_kernel<N, DT, C::rows, C::stages, C::nt, C::p, C::u, C::ctas, QT, false>;
    static std::atomic<uint64_t> attr_done_flat{0};
    if (!ensure_smem_attr(kern, smem, flat ? attr_done_flat : attr_done, dev)) return HADACORE_ERR_CUDA;
    RowGrid gs = g;
    CUtensorMap tin{};
    if (flat) {
      gs.flat_in = static_cast<const uint16_t*>(in);
    } else if (L.in_si == N || L.m_inner == 1) {  // inner rows contiguous: per-outer-block bulk copies
      gs.rows_in = static_cast<const uint16_t*>(in);
      gs.in_so = L.in_so;
    } else if (!encode_small_map(&tin, in, L, L.in_so, L.in_si, N, g)) {
      return HADACORE_ERR_CUDA;
    }
    if (launch_pdl(kern, grid, (C::nt + 1) * 32, smem, stream, tin, static_cast<uint16_t*>(out), out_q, row_scale, gs,
                   s_res) != cudaSuccess)
      return HADACORE_ERR_CUDA;
  } else {
    auto kern = fwht_rows_kernel<N, DT, C::rows, C::stages, C::nt, C::p, C::u, C::ctas, QT>;
    if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
    CUtensorMap tin, tout;
    if (!encode_rows_map(&tin, in, L, L.in_so, L.in_si, N, g, seg) ||
        !encode_rows_map(&tout, QT >= 0 ? in : out, L, QT >= 0 ? L.in_so : L.out_so, QT >= 0 ? L.in_si : L.out_si, N,
                         g, seg))  // the output map is unused when quantizing
      return HADACORE_ERR_CUDA;
    if (launch_pdl(kern, grid, (C::nt + 1) * 32, smem, stream, tin, tout, static_cast<uint16_t*>(out), out_q,
                   row_scale, g, s_res) != cudaSuccess)
      return HADACORE_ERR_CUDA;
  }
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

template <int N, int DT, int QT = QT_NONE>
hadacore_status_t launch_small(const void* in, void* out, int64_t m, float scale, cudaStream_t stream,
                               uint8_t* out_q = nullptr, float* row_scale = nullptr) {
  using T = std::conditional_t<(QT >= 0), TunedSQ<N>, TunedS<N>>;
  constexpr int tile = T::tkb * 1024;
  constexpr int smem = T::st * (tile + small_code_stage_bytes<N, QT, false, tile>()) + int(sizeof(SchedCtl)) + 2 * T::st * 8;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  auto kern = fwht_small_kernel<N, DT, tile, T::st, T::nt, T::u, QT>;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  const int64_t total = m * N * 2;
  const int64_t tiles = (total + tile - 1) / tile;
  const int64_t max_ctas = kClc ? int64_t(INT32_MAX) : int64_t(sm_count(dev));
  const int grid = int(tiles < max_ctas ? tiles : max_ctas);
  if (launch_pdl(kern, grid, (T::nt + 1) * 32, smem, stream, static_cast<const uint16_t*>(in),
                 static_cast<uint16_t*>(out), total, tiles, scale, out_q, row_scale, CUtensorMap{}, CUtensorMap{},
                 RowGrid{}) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

// Row grids with n = 8..64 (hadacore_fwht_strided): 3-D TMA boxes (n, bi, bo) of up to one
// 32 KiB stage; TMA box dims are capped at 256.
template <int N, int DT, int QT = QT_NONE>
hadacore_status_t launch_small_grid(const void* in, void* out, const Layout& L, float scale, cudaStream_t stream,
                                    uint8_t* out_q = nullptr, float* row_scale = nullptr) {
  using T = std::conditional_t<(QT >= 0), TunedSQ<N>, TunedS<N>>;
  constexpr int tile = T::tkb * 1024;
  // The kernel only needs the tile's bytes in shared memory plus, when quantizing, each
  // row's linear index: when each outer row block is contiguous (inner stride = n, e.g.
  // the Q and K heads of a token), the TMA boxes describe it as pseudo-rows of up to 256
  // elements instead of rows of n (16-byte box rows at n = 8 move slowly), the kernel still
  // transforming rows of n (a pseudo-row holds 2^lp whole rows of one outer block).
  Layout Lk = L;
  int nb = N;  // box row length in elements
  if (L.in_si == N && (QT >= 0 || L.out_si == N) && L.m_inner > 1) {
    const int64_t block_el = L.m_inner * N;
    int pn = 256;
    while (pn > N && block_el % pn != 0) pn /= 2;
    if (pn >= 2 * N) {
      Lk.m_inner = block_el / pn;
      Lk.in_si = pn;
      if (QT < 0) Lk.out_si = pn;
      nb = pn;
    }
  }
  const int tile_rows = tile / (2 * nb);
  constexpr int smem = T::st * (tile + small_code_stage_bytes<N, QT, true, tile>()) + int(sizeof(SchedCtl)) + 2 * T::st * 8;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  auto kern = fwht_small_kernel<N, DT, tile, T::st, T::nt, T::u, QT, true>;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  int bi = 1;
  while (bi * 2 <= tile_rows && bi * 2 <= Lk.m_inner && bi * 2 <= 256) bi *= 2;
  const int bo = tile_rows / bi < 256 ? tile_rows / bi : 256;
  RowGrid g{};
  g.m_outer = Lk.m_outer;
  g.m_inner = Lk.m_inner;
  g.out_so = Lk.out_so;
  g.out_si = Lk.out_si;
  while ((1 << g.lbi) < bi) ++g.lbi;
  g.bo = bo;
  g.nib = (Lk.m_inner + bi - 1) / bi;
  g.num_tiles = ((Lk.m_outer + bo - 1) / bo) * g.nib;
  while ((N << g.lp) < nb) ++g.lp;
  CUtensorMap tin, tout;
  if (!encode_small_map(&tin, in, Lk, Lk.in_so, Lk.in_si, nb, g) ||
      !encode_small_map(&tout, QT >= 0 ? in : out, Lk, QT >= 0 ? Lk.in_so : Lk.out_so, QT >= 0 ? Lk.in_si : Lk.out_si, nb,
                        g))  // the output map is unused when quantizing
    return HADACORE_ERR_CUDA;
  const int64_t box_bytes = int64_t(bi) * bo * 2 * nb;
  const int64_t max_ctas = kClc ? int64_t(INT32_MAX) : int64_t(sm_count(dev));
  const int grid = int(g.num_tiles < max_ctas ? g.num_tiles : max_ctas);
  if (launch_pdl(kern, grid, (T::nt + 1) * 32, smem, stream, static_cast<const uint16_t*>(in),
                 static_cast<uint16_t*>(out), box_bytes, g.num_tiles, scale, out_q, row_scale, tin, tout, g) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

template <int DT, int QT = QT_NONE>
hadacore_status_t dispatch_small_grid(const void* in, void* out, const Layout& L, int64_t n, float scale,
                                      cudaStream_t st, uint8_t* q = nullptr, float* rs = nullptr) {
  switch (n) {
    case 8: return launch_small_grid<8, DT, QT>(in, out, L, scale, st, q, rs);
    case 16: return launch_small_grid<16, DT, QT>(in, out, L, scale, st, q, rs);
    case 32: return launch_small_grid<32, DT, QT>(in, out, L, scale, st, q, rs);
    case 64: return launch_small_grid<64, DT, QT>(in, out, L, scale, st, q, rs);
    default: return HADACORE_ERR_INVALID_N;
  }
}

template <int DT, int QT = QT_NONE>
hadacore_status_t dispatch_small(const void* in, void* out, int64_t m, int64_t n, float scale, cudaStream_t st,
                                 uint8_t* q = nullptr, float* rs = nullptr) {
  switch (n) {
    case 2: return launch_small<2, DT, QT>(in, out, m, scale, st, q, rs);
    case 4: return launch_small<4, DT, QT>(in, out, m, scale, st, q, rs);
    case 8: return launch_small<8, DT, QT>(in, out, m, scale, st, q, rs);
    case 16: return launch_small<16, DT, QT>(in, out, m, scale, st, q, rs);
    case 32: return launch_small<32, DT, QT>(in, out, m, scale, st, q, rs);
    case 64: return launch_small<64, DT, QT>(in, out, m, scale, st, q, rs);
    default: return HADACORE_ERR_INVALID_N;
  }
}

template <int DT, int QT>
hadacore_status_t dispatch_n(const void* in, void* out, uint8_t* q, float* rs, const Layout& L, int64_t n, float scale,
                             cudaStream_t st) {
  switch (n) {
    case 128: return launch<128, DT, QT>(in, out, q, rs, L, scale, st);
    case 256: return launch<256, DT, QT>(in, out, q, rs, L, scale, st);
    case 512: return launch<512, DT, QT>(in, out, q, rs, L, scale, st);
    case 1024: return launch<1024, DT, QT>(in, out, q, rs, L, scale, st);
    case 2048: return launch<2048, DT, QT>(in, out, q, rs, L, scale, st);
    case 4096: return launch<4096, DT, QT>(in, out, q, rs, L, scale, st);
    case 8192: return launch<8192, DT, QT>(in, out, q, rs, L, scale, st);
    case 16384: return launch<16384, DT, QT>(in, out, q, rs, L, scale, st);
    case 32768: return launch<32768, DT, QT>(in, out, q, rs, L, scale, st);
    default: return HADACORE_ERR_INVALID_N;
  }
}

Layout contiguous(int64_t m, int64_t n) { return Layout{m, 1, n, n, n, n}; }

// hadacore_fwht / hadacore_fwht_host / hadacore_fwht_quant: n = 2..2^15 (n < 128: NEXT-2,
// fwht_small_kernel); the strided entry points: n = 8..2^15 (rows of >= 16 bytes, TMA).
bool valid_n(int64_t n) { return n >= 2 && n <= 32768 && (n & (n - 1)) == 0; }

size_t elem_size(int dtype) { return dtype == HADACORE_F32 ? 4 : 2; }

// SPEC S:57 (TransformOptions): scale > 0 and finite.  A zero scale would also break
// the fused quantization's contract (row_scale = 1 and zero codes for y == 0): its fast
// path decides on the pre-scale row maximum.
bool valid_scale(float scale) { return std::isfinite(scale) && scale > 0.f; }

template <int N>
hadacore_status_t launch_f32(const void* in, void* out, int64_t m, float scale, cudaStream_t stream) {
  constexpr int rows = N >= 4096 ? 1 : 4096 / N;  // >= 16 KiB of rows per CTA iteration
  constexpr int smem = rows * N * 4;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  auto kern = fwht_f32_kernel<N, rows>;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  const int64_t groups = (m + rows - 1) / rows;
  const int64_t cap = int64_t(sm_count(dev)) * 2;
  if (launch_pdl(kern, int(groups < cap ? groups : cap), 512, smem, stream, static_cast<const float*>(in),
                 static_cast<float*>(out), m, scale) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

// Full-speed fp32 path (NEXT-2, fwht_f32_fast_kernel): 8 consumer warps, 32 KiB
// tiles in a 4-stage ring (64 KiB x 3 for n = 2^14); n = 2^15 = two 2^14 halves +
// f32_half_butterfly_kernel.
#ifndef HC_F32_BIG_N
#define HC_F32_BIG_N 8192  // smallest n with 64 KiB x 3 tiles (n = 8192: 6.33-6.58 -> 6.82-6.84 TB/s, profiles/r02_f32_tiles_ab.txt)
#endif
template <int N> struct TunedF {
  static constexpr int nt = 8, tkb = N >= HC_F32_BIG_N ? 64 : 32, st = N >= HC_F32_BIG_N ? 3 : 4;
};

template <int N>
hadacore_status_t launch_f32_fast(const void* in, void* out, int64_t m, float scale, cudaStream_t stream) {
  using T = TunedF<N>;
  constexpr int tile = T::tkb * 1024;
  constexpr int smem = T::st * tile + int(sizeof(SchedCtl)) + 2 * T::st * 8;
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  auto kern = fwht_f32_fast_kernel<N, tile, T::st, T::nt>;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  const int64_t total = m * N * 4;
  const int64_t tiles = (total + tile - 1) / tile;
  const int64_t max_ctas = kClc ? int64_t(INT32_MAX) : int64_t(sm_count(dev));
  const int grid = int(tiles < max_ctas ? tiles : max_ctas);
  if (launch_pdl(kern, grid, (T::nt + 1) * 32, smem, stream, static_cast<const float*>(in), static_cast<float*>(out),
                 total, tiles, scale) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

hadacore_status_t launch_f32_32k(const void* in, void* out, int64_t m, float scale, cudaStream_t stream) {
#if !defined(HC_F32_TWO_PASS) && !defined(HC_F32_PAIR) && !defined(HC_F32_MC)
  // default: one CTA per SM, the row streamed through a ring of chunk slots
  // (fwht_f32_ring_kernel)
#ifndef HC_RING_CH
#define HC_RING_CH 2048
#endif
#ifndef HC_RING_NT
#define HC_RING_NT 16
#endif
#ifndef HC_RING_DIRECT
#define HC_RING_DIRECT 1
#endif
#ifndef HC_F32_STREAM
#define HC_F32_STREAM 1  // fwht_f32_stream_kernel (chunks released as soon as read); 0: fwht_f32_ring_kernel
#endif
#ifndef HC_STREAM_CH
#define HC_STREAM_CH 16384
#endif
#if HC_F32_STREAM
#ifndef HC_STREAM_NT
#define HC_STREAM_NT 16
#endif
  constexpr int ch = HC_STREAM_CH, nt = HC_STREAM_NT;
  constexpr int slots = (227 * 1024 - 256) / (ch * 4);
  constexpr int smem = slots * ch * 4 + int(sizeof(SchedCtl)) + 2 * slots * 8;
  auto kern = fwht_f32_stream_kernel<ch, slots, nt>;
#else
  constexpr int ch = HC_RING_CH, nt = HC_RING_NT;
  constexpr int slots = (227 * 1024 - 256) / (ch * 4) < 2 * (32768 / ch) - 1 ? (227 * 1024 - 256) / (ch * 4)
                                                                              : 2 * (32768 / ch) - 1;
  constexpr int smem = slots * ch * 4 + (slots + 1) * 8;
  auto kern = fwht_f32_ring_kernel<ch, slots, nt, bool(HC_RING_DIRECT)>;
#endif
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  // fwht_f32_stream_kernel: one CTA per row under CLC (resident CTAs take over the rest);
  // fwht_f32_ring_kernel: a persistent grid with static rows
  const int64_t cap = (HC_F32_STREAM && kStreamClc) ? int64_t(INT32_MAX) : int64_t(sm_count(dev));
  const int64_t ctas = m < cap ? m : cap;
  if (launch_pdl(kern, int(ctas), (nt + 1) * 32, smem, stream, static_cast<const float*>(in),
                 static_cast<float*>(out), m, scale) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
#elif !defined(HC_F32_TWO_PASS)
  // one launch of 2-CTA clusters, a row per cluster: fwht_f32_pair_kernel (DSMEM exchange of
  // the transformed halves; default) or fwht_f32_mc_kernel (HC_F32_MC: top bit first,
  // multicast input halves -- measured slower, 3.2-3.6 vs 4.8 TB/s: profiles/r02_f32_mc_ab.txt)
#ifndef HC_F32_MC
#ifndef HC_PAIR_NT
#define HC_PAIR_NT 16
#endif
#ifndef HC_PAIR_G
#define HC_PAIR_G 2
#endif
  constexpr int st = 3, nt = HC_PAIR_NT, groups = HC_PAIR_G;
  constexpr int smem = st * 65536 + 4 * st * 8;
  auto kern = fwht_f32_pair_kernel<st, nt, groups>;
#else
#ifndef HC_MC_SLOTS
#define HC_MC_SLOTS 5
#endif
#ifndef HC_MC_RB
#define HC_MC_RB 1
#endif
  constexpr int st = HC_MC_SLOTS, nt = 8, nrb = HC_MC_RB;
  constexpr int smem = nrb * 65536 + st * 32768 + 2 * st * 8;
  auto kern = fwht_f32_mc_kernel<st, nt, nrb>;
#endif
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  if (!ensure_smem_attr(kern, smem, attr_done, dev)) return HADACORE_ERR_CUDA;
  // co-resident clusters: a cluster's CTAs share a GPC, so not every SM pairs up --
  // a grid with more clusters than fit at once would run a second wave
  static std::atomic<int> max_clusters[kMaxDevices];
  int cap = (dev >= 0 && dev < kMaxDevices) ? max_clusters[dev].load(std::memory_order_relaxed) : 0;
  if (cap <= 0) {
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(2 * (sm_count(dev) / 2));
    q.blockDim = dim3((nt + 1) * 32);
    q.dynamicSmemBytes = size_t(smem);
    if (cudaOccupancyMaxActiveClusters(&cap, kern, &q) != cudaSuccess || cap <= 0) {
      cudaGetLastError();
      cap = sm_count(dev) / 2;
    }
    if (dev >= 0 && dev < kMaxDevices) max_clusters[dev].store(cap, std::memory_order_relaxed);
  }
  const int64_t clusters = m < cap ? m : int64_t(cap);
  if (launch_pdl(kern, int(2 * clusters), (nt + 1) * 32, smem, stream, static_cast<const float*>(in),
                 static_cast<float*>(out), m, scale) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
#else
  // pass 1: I_2 (x) H_2^14 on the two halves of every row (unnormalized), into `out`
  hadacore_status_t rc = launch_f32_fast<16384>(in, out, 2 * m, 1.f, stream);
  if (rc != HADACORE_OK) return rc;
  // pass 2: H_2 (x) I_2^14 across the halves, times scale, in place in `out`
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return HADACORE_ERR_CUDA;
  const int64_t work = m * 4096, cap = int64_t(sm_count(dev)) * 8;
  const int64_t blocks = (work + 255) / 256;
  if (launch_pdl(f32_half_butterfly_kernel, int(blocks < cap ? blocks : cap), 256, 0, stream,
                 static_cast<const float*>(out), static_cast<float*>(out), m, scale) != cudaSuccess)
    return HADACORE_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
#endif
}

hadacore_status_t dispatch_f32(const void* in, void* out, int64_t m, int64_t n, float scale, cudaStream_t st) {
#ifndef HC_F32_SIMPLE
  switch (n) {
    case 2: return launch_f32_fast<2>(in, out, m, scale, st);
    case 4: return launch_f32_fast<4>(in, out, m, scale, st);
    case 8: return launch_f32_fast<8>(in, out, m, scale, st);
    case 16: return launch_f32_fast<16>(in, out, m, scale, st);
    case 32: return launch_f32_fast<32>(in, out, m, scale, st);
    case 64: return launch_f32_fast<64>(in, out, m, scale, st);
    case 128: return launch_f32_fast<128>(in, out, m, scale, st);
    case 256: return launch_f32_fast<256>(in, out, m, scale, st);
    case 512: return launch_f32_fast<512>(in, out, m, scale, st);
    case 1024: return launch_f32_fast<1024>(in, out, m, scale, st);
    case 2048: return launch_f32_fast<2048>(in, out, m, scale, st);
    case 4096: return launch_f32_fast<4096>(in, out, m, scale, st);
    case 8192: return launch_f32_fast<8192>(in, out, m, scale, st);
    case 16384: return launch_f32_fast<16384>(in, out, m, scale, st);
    case 32768: return launch_f32_32k(in, out, m, scale, st);
    default: return HADACORE_ERR_INVALID_N;
  }
#endif
  // HC_F32_SIMPLE builds: the plain shared-memory debug kernel (one barrier per stage)
  switch (n) {
    case 2: return launch_f32<2>(in, out, m, scale, st);
    case 4: return launch_f32<4>(in, out, m, scale, st);
    case 8: return launch_f32<8>(in, out, m, scale, st);
    case 16: return launch_f32<16>(in, out, m, scale, st);
    case 32: return launch_f32<32>(in, out, m, scale, st);
    case 64: return launch_f32<64>(in, out, m, scale, st);
    case 128: return launch_f32<128>(in, out, m, scale, st);
    case 256: return launch_f32<256>(in, out, m, scale, st);
    case 512: return launch_f32<512>(in, out, m, scale, st);
    case 1024: return launch_f32<1024>(in, out, m, scale, st);
    case 2048: return launch_f32<2048>(in, out, m, scale, st);
    case 4096: return launch_f32<4096>(in, out, m, scale, st);
    case 8192: return launch_f32<8192>(in, out, m, scale, st);
    case 16384: return launch_f32<16384>(in, out, m, scale, st);
    case 32768: return launch_f32<32768>(in, out, m, scale, st);
    default: return HADACORE_ERR_INVALID_N;
  }
}

// Shared by both entry points: everything that can be checked without CUDA.
hadacore_status_t validate(const void* in, const void* out, int64_t m, int64_t n, int dtype, float scale,
                           bool device_buffers) {
  if (dtype != HADACORE_F16 && dtype != HADACORE_BF16 && dtype != HADACORE_F32) return HADACORE_ERR_DTYPE;
  if (!valid_n(n)) return HADACORE_ERR_INVALID_N;
  if (m < 0 || m > INT64_MAX / (int64_t(elem_size(dtype)) * n)) return HADACORE_ERR_INVALID_M;
  if (!valid_scale(scale)) return HADACORE_ERR_SCALE;
  if (m == 0) return HADACORE_OK;
  if (!in || !out) return HADACORE_ERR_NULL;
  if (device_buffers && ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u))
    return HADACORE_ERR_MISALIGNED;
  if (in != out) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(in), b = reinterpret_cast<uintptr_t>(out);
    const uintptr_t bytes = uintptr_t(m) * uintptr_t(n) * elem_size(dtype);
    if (a < b + bytes && b < a + bytes) return HADACORE_ERR_OVERLAP;
  }
  return HADACORE_OK;
}

hadacore_status_t run(const void* in, void* out, int64_t m, int64_t n, int dtype, float scale,
                      cudaStream_t st) {
  if (dtype == HADACORE_F32) return dispatch_f32(in, out, m, n, scale, st);
  if (n < 128)
    return dtype == HADACORE_F16 ? dispatch_small<DT_F16>(in, out, m, n, scale, st)
                                 : dispatch_small<DT_BF16>(in, out, m, n, scale, st);
  const Layout L = contiguous(m, n);
  return dtype == HADACORE_F16 ? dispatch_n<DT_F16, QT_NONE>(in, out, nullptr, nullptr, L, n, scale, st)
                               : dispatch_n<DT_BF16, QT_NONE>(in, out, nullptr, nullptr, L, n, scale, st);
}

template <int DT>
hadacore_status_t run_quant_dt(const void* in, uint8_t* q, float* rs, const Layout& L, int64_t n, int qtype,
                               float scale, cudaStream_t st) {
  if (n < 128 && !(L.m_inner == 1 && L.in_so == n)) {  // rows shorter than 128 on a row grid
    switch (qtype) {
      case HADACORE_Q_E4M3: return dispatch_small_grid<DT, QT_E4M3>(in, nullptr, L, n, scale, st, q, rs);
      case HADACORE_Q_INT8: return dispatch_small_grid<DT, QT_INT8>(in, nullptr, L, n, scale, st, q, rs);
      default: return dispatch_small_grid<DT, QT_INT4>(in, nullptr, L, n, scale, st, q, rs);
    }
  }
  if (n < 128) {  // rows shorter than 128 (fwht_small_kernel's fused epilogue)
    switch (qtype) {
      case HADACORE_Q_E4M3: return dispatch_small<DT, QT_E4M3>(in, nullptr, L.m_outer, n, scale, st, q, rs);
      case HADACORE_Q_INT8: return dispatch_small<DT, QT_INT8>(in, nullptr, L.m_outer, n, scale, st, q, rs);
      default: return dispatch_small<DT, QT_INT4>(in, nullptr, L.m_outer, n, scale, st, q, rs);
    }
  }
  switch (qtype) {
    case HADACORE_Q_E4M3: return dispatch_n<DT, QT_E4M3>(in, nullptr, q, rs, L, n, scale, st);
    case HADACORE_Q_INT8: return dispatch_n<DT, QT_INT8>(in, nullptr, q, rs, L, n, scale, st);
    default: return dispatch_n<DT, QT_INT4>(in, nullptr, q, rs, L, n, scale, st);
  }
}

hadacore_status_t run_quant(const void* in, uint8_t* q, float* rs, int64_t m, int64_t n, int dtype, int qtype,
                            float scale, cudaStream_t st) {
  const Layout L = contiguous(m, n);
  return dtype == HADACORE_F16 ? run_quant_dt<DT_F16>(in, q, rs, L, n, qtype, scale, st)
                               : run_quant_dt<DT_BF16>(in, q, rs, L, n, qtype, scale, st);
}

hadacore_status_t run_strided(const void* in, void* out, const Layout& L, int64_t n, int dtype, float scale,
                              cudaStream_t st) {
  if (n < 128)
    return dtype == HADACORE_F16 ? dispatch_small_grid<DT_F16>(in, out, L, n, scale, st)
                                 : dispatch_small_grid<DT_BF16>(in, out, L, n, scale, st);
  return dtype == HADACORE_F16 ? dispatch_n<DT_F16, QT_NONE>(in, out, nullptr, nullptr, L, n, scale, st)
                               : dispatch_n<DT_BF16, QT_NONE>(in, out, nullptr, nullptr, L, n, scale, st);
}

bool ranges_overlap(const void* a, size_t abytes, const void* b, size_t bbytes) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + bbytes && y < x + abytes;
}

}  // namespace
}  // namespace hadacore

using namespace hadacore;

extern "C" hadacore_status_t hadacore_fwht(const void* in, void* out, int64_t m, int64_t n,
                                           hadacore_dtype_t dtype, float scale, hadacore_stream_t stream) {
  const hadacore_status_t v = validate(in, out, m, n, int(dtype), scale, true);
  if (v != HADACORE_OK || m == 0) return v;
  return run(in, out, m, n, int(dtype), scale, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" hadacore_status_t hadacore_fwht_strided(const void* in, void* out, int64_t m_outer, int64_t m_inner,
                                                   int64_t in_stride_outer, int64_t in_stride_inner,
                                                   int64_t out_stride_outer, int64_t out_stride_inner, int64_t n,
                                                   hadacore_dtype_t dtype, float scale, hadacore_stream_t stream) {
  if (dtype != HADACORE_F16 && dtype != HADACORE_BF16) return HADACORE_ERR_DTYPE;
  if (!valid_n(n) || n < 8) return HADACORE_ERR_INVALID_N;  // row grids: rows of >= 16 bytes (TMA)
  if (m_outer < 0 || m_inner < 0 || m_outer > (int64_t(1) << 31) || m_inner > (int64_t(1) << 31))
    return HADACORE_ERR_INVALID_M;
  if (!valid_scale(scale)) return HADACORE_ERR_SCALE;
  if (m_outer == 0 || m_inner == 0) return HADACORE_OK;
  if (!in || !out) return HADACORE_ERR_NULL;
  const Layout L{m_outer, m_inner, in_stride_outer, m_inner > 1 ? in_stride_inner : n, out_stride_outer,
                 m_inner > 1 ? out_stride_inner : n};
  // strides: multiples of 8 elements (16 B, TMA), rows never overlap, extent fits
  auto bad_stride = [&](int64_t so, int64_t si) {
    if (so % 8 || si % 8 || so <= 0 || si <= 0 || so >= (int64_t(1) << 38) || si >= (int64_t(1) << 38)) return true;
    if (m_inner > 1 && si < n) return true;
    if (m_outer > 1 && so < (m_inner - 1) * si + n) return true;
    return false;
  };
  if (bad_stride(L.in_so, L.in_si) || bad_stride(L.out_so, L.out_si)) return HADACORE_ERR_INVALID_M;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) return HADACORE_ERR_MISALIGNED;
  auto extent = [&](int64_t so, int64_t si) { return size_t(((m_outer - 1) * so + (m_inner - 1) * si + n) * 2); };
  if (in == out) {
    if (L.in_so != L.out_so || L.in_si != L.out_si) return HADACORE_ERR_OVERLAP;
  } else if (ranges_overlap(in, extent(L.in_so, L.in_si), out, extent(L.out_so, L.out_si))) {
    return HADACORE_ERR_OVERLAP;
  }
  return run_strided(in, out, L, n, int(dtype), scale, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" hadacore_status_t hadacore_fwht_quant_strided(const void* in, void* out_q, float* row_scale,
                                                         int64_t m_outer, int64_t m_inner, int64_t in_stride_outer,
                                                         int64_t in_stride_inner, int64_t n, hadacore_dtype_t dtype,
                                                         hadacore_qtype_t qtype, float scale,
                                                         hadacore_stream_t stream) {
  if (qtype != HADACORE_Q_E4M3 && qtype != HADACORE_Q_INT8 && qtype != HADACORE_Q_INT4) return HADACORE_ERR_DTYPE;
  if (dtype != HADACORE_F16 && dtype != HADACORE_BF16) return HADACORE_ERR_DTYPE;
  if (!valid_n(n) || n < 8) return HADACORE_ERR_INVALID_N;  // row grids: rows of >= 16 bytes (TMA)
  if (m_outer < 0 || m_inner < 0 || m_outer > (int64_t(1) << 31) || m_inner > (int64_t(1) << 31))
    return HADACORE_ERR_INVALID_M;
  if (!valid_scale(scale)) return HADACORE_ERR_SCALE;
  if (m_outer == 0 || m_inner == 0) return HADACORE_OK;
  if (!in || !out_q || !row_scale) return HADACORE_ERR_NULL;
  const int64_t si = m_inner > 1 ? in_stride_inner : n;
  if (in_stride_outer % 8 || si % 8 || in_stride_outer <= 0 || si <= 0 || in_stride_outer >= (int64_t(1) << 38) ||
      si >= (int64_t(1) << 38) || (m_inner > 1 && si < n) || (m_outer > 1 && in_stride_outer < (m_inner - 1) * si + n))
    return HADACORE_ERR_INVALID_M;
  if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out_q)) & 15u) ||
      (reinterpret_cast<uintptr_t>(row_scale) & 3u))
    return HADACORE_ERR_MISALIGNED;
  const int64_t m = m_outer * m_inner;
  const size_t in_bytes = size_t((m_outer - 1) * in_stride_outer + (m_inner - 1) * si + n) * 2, s_bytes = size_t(m) * 4;
  const size_t q_bytes = size_t(m) * size_t(n) / (qtype == HADACORE_Q_INT4 ? 2 : 1);
  if (ranges_overlap(in, in_bytes, out_q, q_bytes) || ranges_overlap(in, in_bytes, row_scale, s_bytes) ||
      ranges_overlap(out_q, q_bytes, row_scale, s_bytes))
    return HADACORE_ERR_OVERLAP;
  const Layout L{m_outer, m_inner, in_stride_outer, si, n * m_inner, n};  // codes: contiguous [m_outer * m_inner, n]
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dtype == HADACORE_F16
             ? run_quant_dt<DT_F16>(in, static_cast<uint8_t*>(out_q), row_scale, L, n, int(qtype), scale, st)
             : run_quant_dt<DT_BF16>(in, static_cast<uint8_t*>(out_q), row_scale, L, n, int(qtype), scale, st);
}

extern "C" hadacore_status_t hadacore_fwht_quant(const void* in, void* out_q, float* row_scale, int64_t m,
                                                 int64_t n, hadacore_dtype_t dtype, hadacore_qtype_t qtype,
                                                 float scale, hadacore_stream_t stream) {
  if (qtype != HADACORE_Q_E4M3 && qtype != HADACORE_Q_INT8 && qtype != HADACORE_Q_INT4) return HADACORE_ERR_DTYPE;
  if (dtype == HADACORE_F32) return HADACORE_ERR_DTYPE;  // the fused path takes 16-bit inputs
  // validate `in` (and m, n, dtype, scale) exactly like hadacore_fwht, with out = in
  const hadacore_status_t v = validate(in, in, m, n, int(dtype), scale, true);
  if (v != HADACORE_OK || m == 0) return v;
  if (!out_q || !row_scale) return HADACORE_ERR_NULL;
  if ((reinterpret_cast<uintptr_t>(out_q) & 15u) || (reinterpret_cast<uintptr_t>(row_scale) & 3u))
    return HADACORE_ERR_MISALIGNED;
  const size_t in_bytes = size_t(m) * size_t(n) * 2, s_bytes = size_t(m) * 4;
  const size_t q_bytes = size_t(m) * size_t(n) / (qtype == HADACORE_Q_INT4 ? 2 : 1);  // INT4: two codes per byte
  if (ranges_overlap(in, in_bytes, out_q, q_bytes) || ranges_overlap(in, in_bytes, row_scale, s_bytes) ||
      ranges_overlap(out_q, q_bytes, row_scale, s_bytes))
    return HADACORE_ERR_OVERLAP;
  return run_quant(in, static_cast<uint8_t*>(out_q), row_scale, m, n, int(dtype), int(qtype), scale,
                   reinterpret_cast<cudaStream_t>(stream));
}

extern "C" hadacore_status_t hadacore_fwht_host(const void* in_host, void* out_host, int64_t m, int64_t n,
                                                hadacore_dtype_t dtype, float scale, void* workspace,
                                                size_t workspace_bytes, hadacore_stream_t stream) {
  const hadacore_status_t v = validate(in_host, out_host, m, n, int(dtype), scale, false);
  if (v != HADACORE_OK || m == 0) return v;
  const size_t row_bytes = size_t(n) * elem_size(int(dtype));
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15u) || workspace_bytes < 2 * row_bytes)
    return HADACORE_ERR_WORKSPACE;
  // The workspace is cut into NS slots of at most kBlockBytes, one internal stream
  // each; block b goes H2D -> kernel (in place) -> D2H on stream b % NS.  Small blocks
  // and several streams keep both PCIe directions busy (short pipeline fill/drain).
#ifndef HC_HOST_BLOCK_MB
#define HC_HOST_BLOCK_MB 32  // A/B: profiles/r01_ab_host_pipeline.txt
#endif
#ifndef HC_HOST_SLOTS
#define HC_HOST_SLOTS 4
#endif
  constexpr size_t kBlockBytes = size_t(HC_HOST_BLOCK_MB) << 20;
  constexpr int kMaxSlots = HC_HOST_SLOTS;
  // slot offsets stay 16-byte aligned: rows of < 16 bytes (n < 8) go in groups of
  // 16 / row_bytes rows
  const int64_t align_rows = row_bytes >= 16 ? 1 : int64_t(16 / row_bytes);
  int slots = int(workspace_bytes / row_bytes >= size_t(kMaxSlots * align_rows) ? kMaxSlots : 2);
  int64_t rows_per_slot = int64_t((workspace_bytes / size_t(slots)) / row_bytes);
  const int64_t cap_rows = int64_t(kBlockBytes / row_bytes) > 0 ? int64_t(kBlockBytes / row_bytes) : 1;
  if (rows_per_slot > cap_rows) rows_per_slot = cap_rows;
  rows_per_slot -= rows_per_slot % align_rows;
  if (rows_per_slot < align_rows) {
    slots = 1;
    rows_per_slot = workspace_bytes / row_bytes >= size_t(align_rows) ? align_rows : 1;
  }
  cudaStream_t user = reinterpret_cast<cudaStream_t>(stream);
  // internal streams and event: created once per (host thread, device) and kept (ADVICE /
  // creating and destroying 4 streams + 1 event per call cost a few tens of us)
  struct HostPipe {
    cudaStream_t st[kMaxSlots];
    cudaEvent_t ev;
    bool ready;
  };
  thread_local HostPipe pipes[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return HADACORE_ERR_CUDA;
  HostPipe& hp = pipes[dev];
  if (!hp.ready) {
    for (int i = 0; i < kMaxSlots; ++i)
      if (cudaStreamCreateWithFlags(&hp.st[i], cudaStreamNonBlocking) != cudaSuccess) return HADACORE_ERR_CUDA;
    if (cudaEventCreateWithFlags(&hp.ev, cudaEventDisableTiming) != cudaSuccess) return HADACORE_ERR_CUDA;
    hp.ready = true;
  }
  cudaStream_t* st = hp.st;
  cudaEvent_t ev = hp.ev;
  hadacore_status_t rc = HADACORE_OK;
  {
    // order after everything already queued on the caller's stream
    if (cudaEventRecord(ev, user) != cudaSuccess) rc = HADACORE_ERR_CUDA;
    for (int i = 0; i < slots && rc == HADACORE_OK; ++i)
      if (cudaStreamWaitEvent(st[i], ev, 0) != cudaSuccess) rc = HADACORE_ERR_CUDA;
  }
  const uint8_t* src = static_cast<const uint8_t*>(in_host);
  uint8_t* dst = static_cast<uint8_t*>(out_host);
  int64_t b = 0;
  for (int64_t r0 = 0; rc == HADACORE_OK && r0 < m; r0 += rows_per_slot, ++b) {
    const int64_t rows = (m - r0) < rows_per_slot ? (m - r0) : rows_per_slot;
    const size_t bytes = size_t(rows) * row_bytes;
    const int k = int(b % slots);
    uint8_t* ws = static_cast<uint8_t*>(workspace) + size_t(k) * size_t(rows_per_slot) * row_bytes;
    if (cudaMemcpyAsync(ws, src + size_t(r0) * row_bytes, bytes, cudaMemcpyHostToDevice, st[k]) != cudaSuccess) {
      rc = HADACORE_ERR_CUDA;
      break;
    }
    rc = run(ws, ws, rows, n, int(dtype), scale, st[k]);
    if (rc != HADACORE_OK) break;
    if (cudaMemcpyAsync(dst + size_t(r0) * row_bytes, ws, bytes, cudaMemcpyDeviceToHost, st[k]) != cudaSuccess)
      rc = HADACORE_ERR_CUDA;
  }
  for (int i = 0; i < slots; ++i)
    if (cudaStreamSynchronize(st[i]) != cudaSuccess) rc = HADACORE_ERR_CUDA;
  return rc;
}

// ---------------------------------------------------------------- quant lab (NEXT-4)
namespace hadacore {
namespace {
int log2_pow2(int64_t n) {
  int k = 0;
  while ((int64_t(1) << k) < n) ++k;
  return k;
}
int lab_grid(int64_t work_items, int per_block) {
  const int64_t b = (work_items + per_block - 1) / per_block;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const int64_t cap = int64_t(sm_count(dev)) * 16;  // the current device's SMs
  return int(b < 1 ? 1 : (b < cap ? b : cap));
}
}  // namespace
}  // namespace hadacore

extern "C" hadacore_status_t hadacore_fake_quant(const float* in, float* out, float* row_amax, int64_t m, int64_t n,
                                                 hadacore_qtype_t qtype, int per_tensor, hadacore_stream_t stream) {
  if (qtype != HADACORE_Q_E4M3 && qtype != HADACORE_Q_INT8 && qtype != HADACORE_Q_INT4) return HADACORE_ERR_DTYPE;
  if (!valid_n(n)) return HADACORE_ERR_INVALID_N;
  if (m < 0 || m > INT64_MAX / (4 * n)) return HADACORE_ERR_INVALID_M;
  if (m == 0) return HADACORE_OK;
  if (!in || !out || !row_amax) return HADACORE_ERR_NULL;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(row_amax)) & 15u)
    return HADACORE_ERR_MISALIGNED;
  const size_t bytes = size_t(m) * size_t(n) * 4;
  if ((in != out && ranges_overlap(in, bytes, out, bytes)) || ranges_overlap(in, bytes, row_amax, size_t(m) * 4) ||
      ranges_overlap(out, bytes, row_amax, size_t(m) * 4))
    return HADACORE_ERR_OVERLAP;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  lab::row_amax_kernel<<<lab_grid(m, 8), 256, 0, st>>>(in, row_amax, m, n);
  if (per_tensor) lab::tensor_amax_kernel<<<1, 1024, 0, st>>>(row_amax, m);
  const int64_t total = m * n;
  const int g = lab_grid(total, 256 * 8), k = log2_pow2(n);
  if (qtype == HADACORE_Q_E4M3) lab::fake_quant_kernel<lab::LQ_E4M3><<<g, 256, 0, st>>>(in, out, row_amax, total, k);
  else if (qtype == HADACORE_Q_INT8) lab::fake_quant_kernel<lab::LQ_INT8><<<g, 256, 0, st>>>(in, out, row_amax, total, k);
  else lab::fake_quant_kernel<lab::LQ_INT4><<<g, 256, 0, st>>>(in, out, row_amax, total, k);
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

extern "C" hadacore_status_t hadacore_row_sq_error(const float* a, const float* b, double* out, int64_t m, int64_t n,
                                                   hadacore_stream_t stream) {
  if (n < 1) return HADACORE_ERR_INVALID_N;
  if (m < 0 || m > INT64_MAX / (4 * n)) return HADACORE_ERR_INVALID_M;
  if (m == 0) return HADACORE_OK;
  if (!a || !b || !out) return HADACORE_ERR_NULL;
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 3u ||
      reinterpret_cast<uintptr_t>(out) & 7u)
    return HADACORE_ERR_MISALIGNED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  lab::row_sq_error_kernel<<<lab_grid(m, 8), 256, 0, st>>>(a, b, out, m, n);
  return cudaPeekAtLastError() == cudaSuccess ? HADACORE_OK : HADACORE_ERR_CUDA;
}

extern "C" const char* hadacore_status_string(hadacore_status_t s) {
  switch (s) {
    case HADACORE_OK: return "ok";
    case HADACORE_ERR_INVALID_N:
      return "n must be a power of two in [2, 32768] ([8, 32768] for the strided entry points)";
    case HADACORE_ERR_INVALID_M: return "m must be >= 0 and m*n*2 must fit in int64";
    case HADACORE_ERR_NULL: return "in/out must be non-NULL when m > 0";
    case HADACORE_ERR_MISALIGNED: return "in/out must be 16-byte aligned";
    case HADACORE_ERR_OVERLAP: return "in and out partially overlap (only in == out is allowed)";
    case HADACORE_ERR_DTYPE: return "unsupported dtype / qtype for this entry point";
    case HADACORE_ERR_SCALE: return "scale must be finite and > 0";
    case HADACORE_ERR_CUDA: return "CUDA error (see cudaGetLastError)";
    case HADACORE_ERR_WORKSPACE: return "workspace NULL, misaligned or smaller than two rows";
  }
  return "unknown status";
}

extern "C" int hadacore_version(void) { return kVersion; }

#ifdef HC_TRACE
extern "C" int hadacore_trace_read(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace)) == cudaSuccess ? 0 : 1;
}
extern "C" int hadacore_span_read(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, g_span, bytes < sizeof(g_span) ? bytes : sizeof(g_span)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int hadacore_launches_per_call(int64_t m, int64_t n) {
  return (m > 0 && valid_n(n)) ? 1 : 0;
}

extern "C" int hadacore_launches_per_call_dtype(int64_t m, int64_t n, hadacore_dtype_t dtype) {
#ifndef HC_F32_SIMPLE
#ifdef HC_F32_TWO_PASS
  if (dtype == HADACORE_F32 && m > 0 && n == 32768) return 2;  // two passes (fwht_f32.cuh)
#endif
#endif
  return hadacore_launches_per_call(m, n);
}
