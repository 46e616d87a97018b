// Device engine of the T2C path: TileEngineT2C (reference engine.hpp:311-551) with its state in
// B200 HBM, behind the C ABI of include/splbm_b200.h.
//
// Life cycle: create() builds the tile map on the host (bit-exact, tiling.cpp), uploads the
// tile node types and the 27-neighbour table, derives the per-node gather words on the device
// and allocates the two PDF copies. step() enqueues fused step kernels on the engine stream
// (batches are replayed from cached CUDA graphs) and reads back one 8-byte failure stamp per
// batch. fields() assembles the raster FieldData frame on the device and copies it to the caller.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "mrt.h"
#include "mrt_jit.h"
#include "nccl_api.h"
#include "tiling.h"
#include "tiling_gpu.h"

using namespace splbm_host;

namespace splbm_host {
thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace splbm_host

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(SPLBM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw Error(SPLBM_ERR_CUDA, std::string(what) + " failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
}

// Driver stream memory operations (GPU-side waits/writes on 64-bit flags), resolved through the
// runtime's driver entry point so the library needs no link-time libcuda dependency.
struct StreamMemOps {
  CUresult (*wait)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
  CUresult (*write)(CUstream, CUdeviceptr, cuuint64_t, unsigned int) = nullptr;
};

const StreamMemOps& stream_mem_ops() {
  static StreamMemOps ops;
  static bool done = false;
  if (!done) {
    cudaDriverEntryPointQueryResult q1, q2;
    void* w = nullptr;
    void* v = nullptr;
    CK(cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q1));
    CK(cudaGetDriverEntryPoint("cuStreamWriteValue64", &v, cudaEnableDefault, &q2));
    if (!w || !v || q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess)
      throw Error(SPLBM_ERR_CUDA, "stream memory operations unavailable");
    ops.wait = reinterpret_cast<decltype(ops.wait)>(w);
    ops.write = reinterpret_cast<decltype(ops.write)>(v);
    done = true;
  }
  return ops;
}

constexpr uint64_t kChunkNodes = 1ull << 22;  // initialize_arrays staging (4 x 32 MB)
constexpr int kGraphSteps = 32;               // steps per captured graph (even)
constexpr int kResidentSteps = 1024;          // steps per resident-kernel launch (small domains)

// Resident multi-step kernels are cooperative grids that spin at grid barriers: two of them
// running at once on one device could each hold SMs the other's unscheduled CTAs need. Every
// resident launch in the process waits for the previous one on the same device (one event per
// device), so at most one is in flight.
std::mutex g_resident_mu;
std::map<int, cudaEvent_t> g_resident_last;

}  // namespace

struct splbm_dev_engine {
  // configuration
  int d = 3, q = 19, a = 4, n_tn = 64, periodic = 0, incompressible = 0, device = 0;
  double tau = 1.0, inv_tau = 1.0;
  splbm_dev::BcParams bc{0, 0, 0, 1};
  TileMap tm;  // global tile cover (GPU-built engines: vectors filled on first use, host_tm())
  splbm_dev::TileBuildOut tb;  // GPU tile builder outputs not yet downloaded into tm
  uint64_t tb_bytes = 0;
  // slab (stored = [low halo][owned][high halo], each in compact order)
  int slab_axis = 2, slab_z0 = 0, slab_z1 = 0;
  uint64_t n_low = 0, n_own = 0, n_high = 0, n_stored = 0;
  uint64_t g_low0 = 0, g_own0 = 0, g_high0 = 0;  // global index of each group's first tile
  uint64_t send_low_tiles = 0, send_high_tiles = 0;  // tiles of the bottom / top owned plane
  uint64_t fluid_nodes = 0;
  // device state
  cudaStream_t stream = nullptr;
  void* pdf[2] = {nullptr, nullptr};  // PDF copies in the engine's real type (double / float)
  uint32_t* info = nullptr;
  uint32_t* nb = nullptr;
  uint32_t* order = nullptr;  // column traversal order of large whole-domain engines (StepArgs::order)
  int order_block = 0;        // its column edge B in cells (0 = compact order)
  unsigned long long* failed = nullptr;
  long long* step_base = nullptr;
  int* domain_err = nullptr;
  int* halo_dirs = nullptr;  // [0..4] ez=+1 set, [5..9] ez=-1 set (or 3+3 in 2D)
  int n_halo_dirs = 0;
  double* scratch = nullptr;
  uint64_t scratch_count = 0;  // doubles in `scratch`
  double* reduce_buf = nullptr;  // splbm_dev_reduce partials (allocated on first use)
  // device FieldData frame (splbm_dev_fields), built on the first fields() call
  uint32_t* cells = nullptr;            // cell index of each owned tile
  std::vector<uint64_t> layer_first;    // owned tile index of the first tile at layer >= L
  uint8_t* frame = nullptr;             // rho, ux, uy, uz (double) + mask (byte) for one chunk
  uint64_t frame_nodes = 0;             // raster nodes per chunk
  std::vector<double> mrt_K;  // MRT operator (host copy; passed to the kernels by value), empty = BGK
  // the kernels specialised for mrt_K (StepArgs::jit): two-copy step, single-copy phases 1 / 2
  splbm_host::MrtJitKernels mrt_jit;
  bool mrt_jit_ok = false;
  std::string mrt_jit_why;  // why they are not used (diagnostics)
  uint64_t device_bytes = 0;
  uint32_t l2pf = 0;  // step kernel L2 prefetch distance in CTAs (StepArgs::l2pf)
  uint64_t pdl_min_threads = 4ull * 148 * 256;  // StepArgs::pdl_min_threads (SPLBM_PDL_MIN)
  int x2 = 1;         // StepArgs::x2: two nodes per thread, f32 and D2Q9 f64 (SPLBM_X2=0 disables)
  int off32 = 1;      // StepArgs::off32 when the slots fit 32 bits (SPLBM_OFF32=0 disables)
  // resident multi-step batches (small whole-domain two-copy BGK engines, SPLBM_RESIDENT=0 off):
  // res_blocks CTAs of res_threads threads, res_tpc tiles each; 0 = one launch per step
  unsigned res_blocks = 0, res_threads = 0;
  int res_tpc = 0;
  unsigned* res_flags = nullptr;  // res_blocks x 32 epoch words (ResidentArgs::flags)
  unsigned res_epoch = 0;         // resident steps enqueued so far
  // single-copy (AA) propagation: one PDF array (pdf[0]); `read` is then the state parity
  // (0 natural layout, 1 swapped, see t2c_aa_kernel)
  bool aa = false;
  // TileEngineT2C<float> (paper Table 2 f32 rows): PDFs and node arithmetic in float
  bool f32 = false;
  int es = 8;  // bytes per PDF slot
  int read = 0;
  long step_count = 0;
  uint64_t visits = 0;
  uint64_t launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool batch_timed = false;
  long pending_steps = 0;
  std::map<std::pair<int, int>, cudaGraphExec_t> graphs;
  // native slab halo exchange (NCCL point-to-point on a side stream, overlapped with part 2)
  ncclComm_t comm = nullptr;
  int lower_rank = -1, upper_rank = -1;
  double* halo_buf[4] = {nullptr, nullptr, nullptr, nullptr};  // send_low, send_high, recv_low, recv_high
  uint64_t halo_n[4] = {0, 0, 0, 0};                              // doubles in each
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_arrived = nullptr;
  // fused NVLink peer-store halo exchange (splbm_dev_p2p_attach)
  bool p2p = false, peer_part1 = false;
  cudaStream_t side = nullptr;               // p2p: the boundary planes run here, beside the interior
  cudaEvent_t ev_int[2] = {nullptr, nullptr};  // interior(s) + bump done, by step parity
  cudaEvent_t ev_bnd[2] = {nullptr, nullptr};  // boundary planes(s) + flag writes done
  long long* zero_base = nullptr;  // p2p: failure stamps use the absolute step number as `rel`
  unsigned long long* flags = nullptr;  // [0] faces from below arrived, [1] from above (step seq)
  double* peer_pdf_up[2] = {nullptr, nullptr};
  double* peer_pdf_down[2] = {nullptr, nullptr};
  unsigned long long* peer_flags_up = nullptr;
  unsigned long long* peer_flags_down = nullptr;
  uint64_t peer_down_halo0 = 0;  // first high-halo tile of the lower neighbour
  uint64_t peer_down_own0 = 0;   // single copy: first top-plane tile of the lower neighbour
  uint64_t peer_up_own0 = 0;     // single copy: first bottom-plane tile of the upper neighbour
  unsigned long long comm_seq = 0;
  // p2p halo-arrival wait: cuStreamWaitValue64 with CU_STREAM_WAIT_VALUE_FLUSH where the device
  // can flush remote writes (CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES), else the acquire-polling
  // wait_flags_kernel; SPLBM_P2P_WAIT=kernel|flush forces one (flush must be supported)
  bool wait_flush = false;
  std::vector<void*> ipc_opened;
  std::vector<int> peer_enabled;  // devices this engine's device enabled peer access to

  ~splbm_dev_engine() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (flags) cudaFree(flags);
    if (comm) nccl().CommDestroy(comm);
    for (double* b : halo_buf)
      if (b) cudaFree(b);
    if (ev_packed) cudaEventDestroy(ev_packed);
    if (ev_arrived) cudaEventDestroy(ev_arrived);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (side) cudaStreamSynchronize(side);
    for (int k = 0; k < 2; ++k) {
      if (ev_int[k]) cudaEventDestroy(ev_int[k]);
      if (ev_bnd[k]) cudaEventDestroy(ev_bnd[k]);
    }
    if (side) cudaStreamDestroy(side);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    splbm_dev::free_tile_build(&tb);
    for (void* p : {static_cast<void*>(pdf[0]), static_cast<void*>(pdf[1]),
                    static_cast<void*>(info), static_cast<void*>(nb), static_cast<void*>(failed),
                    static_cast<void*>(step_base), static_cast<void*>(domain_err),
                    static_cast<void*>(zero_base),
                    static_cast<void*>(halo_dirs), static_cast<void*>(scratch),
                    static_cast<void*>(reduce_buf), static_cast<void*>(order),
                    static_cast<void*>(res_flags),
                    static_cast<void*>(cells), static_cast<void*>(frame)})
      if (p) cudaFree(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }

  template <class T>
  T* alloc(std::size_t count) {
    void* p = nullptr;
    const std::size_t bytes = std::max<std::size_t>(count, 1) * sizeof(T);
    const cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess)
      throw Error(SPLBM_ERR_CUDA, "cudaMalloc of " + std::to_string(bytes) +
                                      " bytes failed: " + cudaGetErrorString(e));
    device_bytes += bytes;
    return static_cast<T*>(p);
  }

  uint64_t tile_stride() const { return static_cast<uint64_t>(q) * n_tn; }
  void* cur_pdf() const { return aa ? pdf[0] : pdf[read]; }
  splbm_dev::StateView view() const { return {nb, a, aa && read == 1 ? 1 : 0}; }

  splbm_dev::StepArgs step_args(int rd, int rel) const {
    splbm_dev::StepArgs s{};
    s.read = aa ? pdf[0] : pdf[rd];
    s.write = aa ? pdf[0] : pdf[1 - rd];
    s.aa = aa ? 1 + rd : 0;
    s.info = info;
    s.nb = nb;
    s.t0 = n_low;
    s.n_nodes = n_own * n_tn;
    s.skip_at = UINT64_MAX;
    s.skip_by = 0;
    s.a = a;
    s.inv_tau = inv_tau;
    s.mrt_K = mrt_K.empty() ? nullptr : mrt_K.data();
    s.bc = bc;
    s.failed = failed;
    s.step_base = step_base;
    s.rel = rel;
    if (p2p && zero_base) {  // steps enqueued one by one (no graphs): absolute step, no bump
      s.step_base = zero_base;
      s.rel = static_cast<int>(step_count) + rel;
    }
    s.l2pf = l2pf;
    s.pdl_min_threads = pdl_min_threads;
    s.x2 = x2;
    s.off32 = off32 && n_stored * tile_stride() < (1ull << 32);
    s.order = order;
    s.jit = !mrt_jit_ok ? nullptr : (aa ? mrt_jit.aa[rd] : mrt_jit.step);
    if (peer_part1 && aa) {  // single copy: phase 1 reads/writes the halo nodes' slots in place
      if (rd == 0) {
        s.peer_down = peer_pdf_down[0] ? peer_pdf_down[0] + peer_down_own0 * tile_stride() : nullptr;
        s.peer_up = peer_pdf_up[0] ? peer_pdf_up[0] + peer_up_own0 * tile_stride() : nullptr;
        s.halo_lo_end = n_low;
        s.halo_hi_begin = n_low + n_own;
      }
    } else if (peer_part1) {
      s.peer_up = peer_pdf_up[1 - rd];
      s.peer_down = peer_pdf_down[1 - rd] ? peer_pdf_down[1 - rd] + peer_down_halo0 * tile_stride() : nullptr;
      s.top_begin = n_low + n_own - send_high_tiles;
      s.bot_begin = n_low;
      s.bot_end = n_low + send_low_tiles;
    }
    return s;
  }

  // One step's kernel over the stored tile range [t_begin, t_end) from copy rd (no flip).
  void launch_range(int rd, uint64_t t_begin, uint64_t t_end) {
    if (t_end <= t_begin) return;
    splbm_dev::StepArgs s = step_args(rd, 0);
    s.order = nullptr;  // (slab parts: compact ranges)
    s.t0 = t_begin;
    s.n_nodes = (t_end - t_begin) * n_tn;
    CK(splbm_dev::launch_step(d, incompressible != 0, f32, s, stream));
    ++launches;
  }

  // Slab-overlap parts: 1 = the bottom and top owned planes (their faces are exchanged while
  // part 2, the interior planes, runs); part 2 then swaps the copies and counts the step.
  void step_part(int part, cudaEvent_t before_bump = nullptr) {
    const uint64_t b0 = n_low, b1 = n_low + send_low_tiles;          // bottom plane
    const uint64_t t0 = n_low + n_own - send_high_tiles, t1 = n_low + n_own;  // top plane
    const bool merged = b1 >= t0;  // one or two planes: the boundary covers the whole slab
    if (part == 1) {
      if (merged) {
        launch_range(read, b0, t1);
      } else if (b1 > b0 && t1 > t0) {  // both planes in one launch, jumping the interior
        splbm_dev::StepArgs s = step_args(read, 0);
        s.order = nullptr;
        s.t0 = b0;
        s.n_nodes = (send_low_tiles + send_high_tiles) * n_tn;
        s.skip_at = send_low_tiles;
        s.skip_by = t0 - b1;
        CK(splbm_dev::launch_step(d, incompressible != 0, f32, s, stream));
        ++launches;
      } else {
        launch_range(read, b0, b1);
        launch_range(read, t0, t1);
      }
      return;
    }
    if (!merged) launch_range(read, b1, t0);
    if (before_bump) CK(cudaStreamWaitEvent(stream, before_bump, 0));
    CK(splbm_dev::launch_bump(step_base, 1, stream));
    ++launches;
    read = 1 - read;
    ++step_count;
    visits += n_own;
  }

  // Face pack / unpack on the engine stream (see splbm_dev_halo_pack / _unpack for the layout).
  void halo_copy(int copy, uint64_t tile0, uint64_t ntiles, int layer, const int* dirs, double* buf,
                 bool pack, bool mask = false) {
    if (f32) throw config_error("slab halo exchange is built for the f64 engine");
    if (!ntiles || !buf) return;
    splbm_dev::HaloArgs h{static_cast<double*>(aa ? pdf[0] : pdf[copy]), buf, tile0, ntiles, a, layer,
                          n_halo_dirs, dirs, pack ? 1 : 0, mask ? info : nullptr};
    CK(splbm_dev::launch_halo(d, h, stream));
    ++launches;
  }
  void pack_faces(int copy, double* low, double* high) {
    halo_copy(copy, n_low, send_low_tiles, 0, halo_dirs + n_halo_dirs, low, true);
    halo_copy(copy, n_low + n_own - send_high_tiles, send_high_tiles, a - 1, halo_dirs, high, true);
  }
  void unpack_faces(int copy, double* low, double* high) {
    halo_copy(copy, 0, n_low, a - 1, halo_dirs, low, false);
    halo_copy(copy, n_low + n_own, n_high, 0, halo_dirs + n_halo_dirs, high, false);
  }
  // Single copy, after a phase-1 step: the halo slots my scatter wrote go back to their owners
  // (low halo, top layer, upward dirs -> lower rank; high halo, bottom layer, downward dirs ->
  // upper rank), and the owners store only the slots whose downstream node is non-solid.
  void pack_back(double* low, double* high) {
    if (!aa) throw config_error("the backward face exchange is the single-copy scheme's");
    halo_copy(0, 0, n_low, a - 1, halo_dirs, low, true);
    halo_copy(0, n_low + n_own, n_high, 0, halo_dirs + n_halo_dirs, high, true);
  }
  void unpack_back(double* low, double* high) {
    if (!aa) throw config_error("the backward face exchange is the single-copy scheme's");
    halo_copy(0, n_low, send_low_tiles, 0, halo_dirs + n_halo_dirs, low, false, true);
    halo_copy(0, n_low + n_own - send_high_tiles, send_high_tiles, a - 1, halo_dirs, high, false, true);
  }

  // One step of the multi-GPU slab mode: boundary planes, pack their faces, NCCL send/recv on the
  // comm stream (one group, order [send up, recv below, send down, recv above] as
  // slab.HaloExchange), interior planes overlapping the transfer, then unpack into the halo planes.
  void exchange_step() {
    step_part(1);
    const int next = 1 - read;
    pack_faces(next, lower_rank >= 0 ? halo_buf[0] : nullptr, upper_rank >= 0 ? halo_buf[1] : nullptr);
    CK(cudaEventRecord(ev_packed, stream));
    CK(cudaStreamWaitEvent(comm_stream, ev_packed, 0));
    const NcclApi& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    if (upper_rank >= 0 && halo_n[1])
      nccl_check(N.Send(halo_buf[1], halo_n[1], ncclFloat64, upper_rank, comm, comm_stream), "ncclSend");
    if (lower_rank >= 0 && halo_n[2])
      nccl_check(N.Recv(halo_buf[2], halo_n[2], ncclFloat64, lower_rank, comm, comm_stream), "ncclRecv");
    if (lower_rank >= 0 && halo_n[0])
      nccl_check(N.Send(halo_buf[0], halo_n[0], ncclFloat64, lower_rank, comm, comm_stream), "ncclSend");
    if (upper_rank >= 0 && halo_n[3])
      nccl_check(N.Recv(halo_buf[3], halo_n[3], ncclFloat64, upper_rank, comm, comm_stream), "ncclRecv");
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    CK(cudaEventRecord(ev_arrived, comm_stream));
    step_part(2);
    CK(cudaStreamWaitEvent(stream, ev_arrived, 0));
    unpack_faces(read, lower_rank >= 0 ? halo_buf[2] : nullptr, upper_rank >= 0 ? halo_buf[3] : nullptr);
  }

  // One slab step with the faces stored by the boundary-plane kernel straight into the neighbours'
  // halo tiles (NVLink peer stores). Stream-ordered flags: before the boundary planes of step
  // seq+1 wait until both neighbours finished their boundary planes of step seq (so my halos hold
  // their faces and they no longer read the halo copy I am about to overwrite); afterwards publish
  // seq+1 into the neighbours' flags.
  //
  // The boundary planes run on a side stream, concurrently with the interior planes of the same
  // step on the engine stream (SURVEY §8e overlap): step s with parity k
  //   side:   wait ev_int[k^1] (interior(s-1): the planes read what it wrote next to them, and
  //           overwrite the copy it read) -> flag waits -> boundary planes (+ peer stores) -> flag
  //           writes -> record ev_bnd[k]
  //   engine: wait ev_bnd[k^1] (boundary(s-1), same reasons) -> interior(s) -> record ev_int[k]
  // Failure stamps carry the absolute step number (no bump kernel between the parts).
  void p2p_step() {
    const StreamMemOps& ops = stream_mem_ops();
    const int k = static_cast<int>(comm_seq & 1);
    CK(cudaStreamWaitEvent(side, ev_int[k ^ 1], 0));
    const unsigned long long* f_below = peer_pdf_down[0] ? &flags[0] : nullptr;
    const unsigned long long* f_above = peer_pdf_up[0] ? &flags[1] : nullptr;
    if (wait_flush) {  // GPU front-end wait + flush of outstanding remote writes
      for (const unsigned long long* f : {f_below, f_above})
        if (f)
          cu_check(ops.wait(side, reinterpret_cast<CUdeviceptr>(f), comm_seq,
                            CU_STREAM_WAIT_VALUE_GEQ | CU_STREAM_WAIT_VALUE_FLUSH),
                   "cuStreamWaitValue64");
    } else if (f_below || f_above) {  // system-scope acquire polling (wait_flags_kernel)
      CK(splbm_dev::launch_wait_flags(f_below, f_above, comm_seq, side));
      ++launches;
    }
    peer_part1 = true;
    std::swap(stream, side);  // part 1 launches on the side stream
    step_part(1);
    std::swap(stream, side);
    peer_part1 = false;
    ++comm_seq;
    if (peer_pdf_up[0])  // the upper rank's "from below" flag
      cu_check(ops.write(side, reinterpret_cast<CUdeviceptr>(&peer_flags_up[0]), comm_seq, CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
    if (peer_pdf_down[0])  // the lower rank's "from above" flag
      cu_check(ops.write(side, reinterpret_cast<CUdeviceptr>(&peer_flags_down[1]), comm_seq, CU_STREAM_WRITE_VALUE_DEFAULT), "cuStreamWriteValue64");
    CK(cudaEventRecord(ev_bnd[k], side));
    CK(cudaStreamWaitEvent(stream, ev_bnd[k ^ 1], 0));
    const uint64_t b1 = n_low + send_low_tiles, t0 = n_low + n_own - send_high_tiles;
    if (b1 < t0) launch_range(read, b1, t0);  // interior planes
    CK(cudaEventRecord(ev_int[k], stream));
    read = 1 - read;
    ++step_count;
    visits += n_own;
  }

  // Enqueue k steps starting from parity rd (direct launches) + the counter bump.
  void enqueue_direct(int rd, int k) {
    for (int r = 0; r < k; ++r) {
      CK(splbm_dev::launch_step(d, incompressible != 0, f32, step_args(rd, r), stream));
      rd = 1 - rd;
      ++launches;
    }
    CK(splbm_dev::launch_bump(step_base, k, stream));
    ++launches;
  }

  // k steps from parity rd in one resident launch (+ the counter bump), serialised per device.
  void enqueue_resident(int rd, int k) {
    splbm_dev::ResidentArgs ra{};
    ra.s = step_args(rd, 0);
    ra.pdf0 = pdf[0];
    ra.pdf1 = pdf[1];
    ra.rd0 = rd;
    ra.nsteps = k;
    ra.tiles_per_cta = res_tpc;
    ra.flags = res_flags;
    ra.epoch0 = res_epoch;
    res_epoch += static_cast<unsigned>(k);
    {
      std::lock_guard<std::mutex> lk(g_resident_mu);
      cudaEvent_t& last = g_resident_last[device];
      if (last) CK(cudaStreamWaitEvent(stream, last, 0));
      else CK(cudaEventCreateWithFlags(&last, cudaEventDisableTiming));
      CK(splbm_dev::launch_resident(d, incompressible != 0, f32, ra, res_blocks, res_threads, stream));
      CK(cudaEventRecord(last, stream));
    }
    CK(splbm_dev::launch_bump(step_base, k, stream));
    launches += 2;
  }

  cudaGraphExec_t graph_for(int rd) {
    const auto key = std::make_pair(kGraphSteps, rd);
    auto it = graphs.find(key);
    if (it != graphs.end()) return it->second;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    const uint64_t saved = launches;
    try {
      enqueue_direct(rd, kGraphSteps);
    } catch (...) {
      cudaStreamEndCapture(stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    launches = saved;
    CK(cudaStreamEndCapture(stream, &g));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    graphs[key] = ex;
    return ex;
  }

  void enqueue_steps(long n) {
    if (comm) {  // slab mode with a native communicator: every step exchanges faces
      for (long k = 0; k < n; ++k) exchange_step();
      return;
    }
    if (p2p) {  // slab mode with NVLink peer stores
      // the first waits of both streams: everything enqueued on the engine stream so far
      CK(cudaEventRecord(ev_int[(comm_seq & 1) ^ 1], stream));
      CK(cudaEventRecord(ev_bnd[(comm_seq & 1) ^ 1], stream));
      for (long k = 0; k < n; ++k) p2p_step();
      CK(cudaStreamWaitEvent(stream, ev_bnd[(comm_seq & 1) ^ 1], 0));  // join the last planes
      CK(splbm_dev::launch_bump(step_base, n, stream));  // keep step_base in step with step_count
      ++launches;
      return;
    }
    long left = n;
    if (res_blocks) {  // small domain: whole batches inside one cooperative grid
      while (left > 0) {
        const int k = static_cast<int>(std::min<long>(left, kResidentSteps));
        enqueue_resident(read, k);
        if (k & 1) read = 1 - read;
        left -= k;
      }
    }
    while (left >= kGraphSteps) {
      CK(cudaGraphLaunch(graph_for(read), stream));
      launches += kGraphSteps + 1;
      left -= kGraphSteps;  // kGraphSteps is even: parity unchanged
    }
    if (left > 0) {
      enqueue_direct(read, static_cast<int>(left));
      if (left & 1) read = 1 - read;
    }
    step_count += n;
    visits += n_own * static_cast<uint64_t>(n);
  }
};

namespace {

splbm_dev_engine* checked(splbm_dev_engine* e) {
  if (!e) throw config_error("null engine");
  CK(cudaSetDevice(e->device));
  return e;
}

void build(splbm_dev_engine* e, const splbm_dev_desc* desc) {
  if (!desc || !desc->types) throw config_error("null descriptor");
  // SPLBM_BUILD_TIMING=1: per-phase wall times of the engine build on stderr
  const bool timing = std::getenv("SPLBM_BUILD_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build] %-16s %8.1f ms\n", name,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  const int d = desc->d;
  if (d != 2 && d != 3) throw config_error("dimension must be 2 or 3");
  if (!(desc->tau > 0.5)) throw config_error("relaxation time tau must be > 0.5");  // collision.cpp:90
  e->d = d;
  e->q = d == 2 ? 9 : 19;
  e->a = desc->tile > 0 ? desc->tile : (d == 2 ? 16 : 4);  // SimConfig::tile_edge (engine.hpp:575)
  e->periodic = desc->periodic;
  e->incompressible = desc->incompressible ? 1 : 0;
  e->tau = desc->tau;
  e->f32 = desc->single_precision != 0;
  e->es = e->f32 ? 4 : 8;
  // inv_tau_ = T(1.0 / tau) (collision.cpp:93); a float value is exact in the double argument
  e->inv_tau = e->f32 ? static_cast<double>(static_cast<float>(1.0 / desc->tau)) : 1.0 / desc->tau;
  if (e->f32 && (desc->slab_z0 != 0 || desc->slab_z1 != 0))
    throw config_error("the f32 engine is a single-GPU engine (no slab)");
  e->bc = {desc->bc_velocity[0], desc->bc_velocity[1], desc->bc_velocity[2], desc->bc_density};
  e->device = desc->device;
  int dims[3] = {desc->dims[0], desc->dims[1], d == 2 ? 1 : desc->dims[2]};
  if (d == 2 && desc->dims[2] != 1 && desc->dims[2] != 0)
    throw config_error("2D geometry requires nz = 1");

  if (desc->single_copy) {  // single PDF array, AA access pattern
    const bool pow2 = e->a == 2 || e->a == 4 || (d == 2 && (e->a == 8 || e->a == 16));
    if (!pow2) throw config_error("single-copy propagation needs a power-of-two tile (a = 2, 4; 2D a <= 16)");
    e->aa = true;
  }
  // ---- device ------------------------------------------------------------------------------
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(SPLBM_ERR_CUDA, "no CUDA device available (the T2C path has no CPU fallback)");
  if (e->device < 0 || e->device >= ndev) throw config_error("invalid CUDA device ordinal");
  CK(cudaSetDevice(e->device));
  {
    // L2 prefetch distance of the step kernel: two CTAs per SM ahead (64-thread CTAs: 296 tiles
    // of a 4^3 3D domain). Interleaved A/B on a B200 against no prefetch: channel 128^3 +6 %,
    // RAS 256^3 +3 %, 2D 4096^2 +8 %; four times farther ahead loses part of it again.
    // SPLBM_L2PF overrides it (0 = off) for tuning sweeps.
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device));
    e->l2pf = static_cast<uint32_t>(2 * sms);
    // single copy: five CTAs per SM ahead (round 2, with 16 phase-1 CTAs per SM: RAS 256^3 phi 0.2
    // / 0.5 -3 % / -1 % per step against four, dense unchanged; six and more cost dense 1 %)
    if (e->aa) e->l2pf = static_cast<uint32_t>(5 * sms);
    if (const char* v = std::getenv("SPLBM_L2PF")) e->l2pf = static_cast<uint32_t>(std::atoi(v));
    if (const char* v = std::getenv("SPLBM_PDL_MIN")) e->pdl_min_threads = std::strtoull(v, nullptr, 10);
    if (const char* v = std::getenv("SPLBM_X2")) e->x2 = std::atoi(v);
    if (const char* v = std::getenv("SPLBM_OFF32")) e->off32 = std::atoi(v);
  }
  phase("device_select");
  CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  const bool slab_mode = desc->slab_z0 != 0 || desc->slab_z1 != 0;
  // Whole-domain engines build the tile map on the GPU (tiling_gpu.cu; SPLBM_HOST_TILES=1 forces
  // the host builder); slab engines use the host builder and its slab tables.
  const bool gpu_tiles = !slab_mode && std::getenv("SPLBM_HOST_TILES") == nullptr;
  TileMap& tm = e->tm;
  SlabLayout sl;
  std::vector<uint32_t> nb_local;
  std::vector<uint8_t> types_local;
  if (gpu_tiles) {
    validate_tiling(d, dims, e->a, e->periodic);
    tm.d = d;
    tm.a = e->a;
    tm.periodic = e->periodic;
    for (int k = 0; k < 3; ++k) tm.dims[k] = dims[k];
    tile_dims(d, dims, e->a, tm.grid_dims, tm.padded_dims);
    tm.n_tn = e->a * e->a * (d == 3 ? e->a : 1);
    const std::size_t n = static_cast<std::size_t>(dims[0]) * dims[1] * dims[2];
    uint8_t* raster_d = nullptr;
    CK(cudaMalloc(&raster_d, n));
    cudaError_t err = cudaMemcpy(raster_d, desc->types, n, cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
      err = splbm_dev::build_tiles_device(raster_d, d, dims, e->a, e->periodic, tm.grid_dims, e->stream, &e->tb);
    cudaFree(raster_d);
    CK(err);
    tm.n_tiles = e->tb.n_tiles;
    e->tb_bytes = tm.n_tiles * (12ull + 2ull * tm.n_tn) +
                  static_cast<uint64_t>(tm.grid_dims[0]) * tm.grid_dims[1] * tm.grid_dims[2] * 4;
    e->device_bytes += e->tb_bytes;
    sl.axis = d == 3 ? 2 : 1;
    sl.z1 = tm.grid_dims[sl.axis];
    sl.n_own = tm.n_tiles;
    e->fluid_nodes = e->tb.fluid_nodes;
    e->n_tn = tm.n_tn;
    phase("gpu_tiles");
    // Column traversal (tiling_gpu.h), an experiment switch: SPLBM_ORDER=BY[xBX] steps the tiles
    // in (x, y) columns of BX x BY cells (BX default: whole rows = row bands), each walked
    // z-major, so a tile's -z neighbour was stepped one column-plane earlier instead of a whole
    // plane (1024^3: ~200 MB per plane, beyond L2). Measured slower than the compact order on
    // every workload tried (DESIGN.md kept/dropped table): off by default.
    if (d == 3 && !e->f32 && (e->a == 2 || e->a == 4) && tm.n_tiles) {
      int BY = 0, BX = 0;
      if (const char* v = std::getenv("SPLBM_ORDER")) {
        BY = std::atoi(v);
        if (const char* x = std::strchr(v, 'x')) BX = std::atoi(x + 1);
      }
      if (BX <= 0) BX = tm.grid_dims[0];
      if (BY > 0 && (BX < tm.grid_dims[0] || BY < tm.grid_dims[1])) {
        e->order = e->alloc<uint32_t>(tm.n_tiles);
        CK(splbm_dev::build_column_order(e->tb.tile_map, tm.grid_dims, BX, BY, tm.n_tiles, e->order,
                                         e->stream));
        e->order_block = BY;
      }
      phase("column_order");
    }
  } else {
    tm = build_tile_map(desc->types, d, dims, e->a, e->periodic);
    phase("tile_map");
    e->n_tn = tm.n_tn;
    const std::vector<uint32_t> nb_global = neighbour_table(tm);
    phase("neighbour_table");
    const std::vector<uint8_t> deg = degenerate_mask(desc->types, d, dims, e->periodic);
    phase("degenerate_mask");
    // ---- slab of tile planes along the last axis -------------------------------
    sl = slab_layout(tm, desc->slab_z0, desc->slab_z1);
    slab_tables(tm, sl, nb_global, deg, nb_local, types_local);
    phase("slab_tables");
    for (uint64_t s = sl.n_low; s < sl.n_low + sl.n_own; ++s) e->fluid_nodes += tm.fluid_count[sl.global_of(s)];
  }

  // PressureBC under the quasi-compressible model needs rho_bc > 0 (lattice.hpp:76-78)
  if (!e->incompressible && !(desc->bc_density > 0.0)) {
    bool has_p = false;
    for (std::size_t i = 0, n = static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]; i < n && !has_p; ++i)
      has_p = desc->types[i] == 3;
    if (has_p) throw domain_error("equilibrium requires rho > 0 for the quasi-compressible model");
  }

  e->slab_axis = sl.axis;
  e->slab_z0 = sl.z0;
  e->slab_z1 = sl.z1;
  e->n_low = sl.n_low;
  e->n_own = sl.n_own;
  e->n_high = sl.n_high;
  e->g_low0 = sl.g_low0;
  e->g_own0 = sl.g_own0;
  e->g_high0 = sl.g_high0;
  e->n_stored = sl.stored();
  e->send_low_tiles = sl.send_low_tiles;
  e->send_high_tiles = sl.send_high_tiles;
  const uint64_t S = e->n_stored;
  const int n_tn = e->n_tn;
  CK(cudaEventCreate(&e->ev0));
  CK(cudaEventCreate(&e->ev1));
  const uint64_t nslots = S * e->tile_stride();
  e->pdf[0] = e->alloc<char>(nslots * e->es);
  if (!e->aa) e->pdf[1] = e->alloc<char>(nslots * e->es);
  e->info = e->alloc<uint32_t>(S * n_tn);
  const int nbs = d == 3 ? 27 : 9;  // 2D keeps only the dz = 0 slice (cells 9..17)
  if (gpu_tiles) {  // the builder's table is already in the device layout
    e->nb = e->tb.nb;
    e->tb.nb = nullptr;
    e->device_bytes += std::max<uint64_t>(S, 1) * nbs * 4;
  } else {
    e->nb = e->alloc<uint32_t>(S * nbs);
  }
  e->failed = e->alloc<unsigned long long>(1);
  e->step_base = e->alloc<long long>(1);
  e->domain_err = e->alloc<int>(1);
  e->scratch_count = std::max<uint64_t>({4 * std::min<uint64_t>(kChunkNodes, std::max<uint64_t>(S * n_tn, 1)),
                                          e->tile_stride(), 8ull * n_tn});
  e->scratch = e->alloc<double>(e->scratch_count);
  if (desc->collision == 1) {  // MRT
    e->mrt_K = mrt_kernel(d, desc->tau, desc->mrt_rates);
    // power-of-two steps (two copies and both single-copy phases) use the kernels specialised for
    // this operator (mrt_jit.cpp); SPLBM_MRT_JIT=0 keeps the generic instantiations
    const char* jit_env = std::getenv("SPLBM_MRT_JIT");
    const bool pow2 = d == 3 ? (e->a == 2 || e->a == 4) : (e->a == 2 || e->a == 4 || e->a == 8 || e->a == 16);
    if (pow2 && !(jit_env && std::atoi(jit_env) == 0)) {
      int loga = 0;
      while ((1 << loga) < e->a) ++loga;
      e->mrt_jit_ok = splbm_host::mrt_jit_kernels(d, loga, e->incompressible != 0, e->f32, e->mrt_K,
                                                  &e->mrt_jit, &e->mrt_jit_why);
    }
  } else if (desc->collision != 0) {
    throw config_error("unknown collision kind");
  }
  // face direction sets: slab axis component +1 then -1 (lattice.cpp order)
  {
    static const int e3z[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
    static const int e2y[9] = {0, 0, 0, 1, -1, 1, -1, -1, 1};
    std::vector<int> dirs;
    for (int sgn : {1, -1})
      for (int i = 0; i < e->q; ++i)
        if ((d == 3 ? e3z[i] : e2y[i]) == sgn) dirs.push_back(i);
    e->n_halo_dirs = static_cast<int>(dirs.size()) / 2;
    e->halo_dirs = e->alloc<int>(dirs.size());
    CK(cudaMemcpy(e->halo_dirs, dirs.data(), dirs.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  CK(cudaMemsetAsync(e->step_base, 0, sizeof(long long), e->stream));
  CK(cudaMemsetAsync(e->pdf[0], 0, nslots * e->es, e->stream));
  if (e->pdf[1]) CK(cudaMemsetAsync(e->pdf[1], 0, nslots * e->es, e->stream));
  if (!gpu_tiles) {
    if (d == 2) {
      std::vector<uint32_t> nb2(S * 9);
      for (uint64_t t = 0; t < S; ++t)
        for (int k = 0; k < 9; ++k) nb2[t * 9 + k] = nb_local[t * 27 + 9 + k];
      nb_local.swap(nb2);
    }
    CK(cudaMemcpyAsync(e->nb, nb_local.data(), nb_local.size() * 4, cudaMemcpyHostToDevice, e->stream));
  }
  {
    // the tile node types (GPU builder output or a host upload) are freed on every exit path
    uint8_t* types_d = e->tb.types_bc;
    if (gpu_tiles) e->tb.types_bc = nullptr;
    std::unique_ptr<uint8_t, cudaError_t (*)(void*)> types_guard(nullptr, cudaFree);
    if (!gpu_tiles) {
      CK(cudaMalloc(&types_d, std::max<std::size_t>(types_local.size(), 1)));
      types_guard.reset(types_d);
      CK(cudaMemcpyAsync(types_d, types_local.data(), types_local.size(), cudaMemcpyHostToDevice, e->stream));
    } else {
      types_guard.reset(types_d);
    }
    splbm_dev::NodeInfoArgs ni{types_d, e->nb, e->info, S, e->a, 32 / e->es};
    CK(splbm_dev::launch_node_info(d, ni, e->stream));
    ++e->launches;
    CK(cudaStreamSynchronize(e->stream));
    types_guard.reset();
    if (gpu_tiles) {
      e->device_bytes -= S * n_tn;
      e->tb_bytes -= S * n_tn;
    }
  }
  phase("device_tables");
  // Resident multi-step batches (t2c_resident_kernel) when the whole domain fits one CTA of at
  // most 1024 threads (512 for D3Q19 f64) per SM: there the launch gap, not HBM, sets the step time.
  {
    int coop = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, e->device));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device));
    const char* env = std::getenv("SPLBM_RESIDENT");
    const bool want = env ? std::atoi(env) != 0 : true;
    // two resident CTAs per SM (half the nodes each) measured 5 % faster than one on configs[0]
    // (a = 4 and 16; three: no further gain); one when two do not fit. SPLBM_RESIDENT_PER_SM overrides.
    const char* per_env = std::getenv("SPLBM_RESIDENT_PER_SM");
    const int first = per_env ? std::max(1, std::atoi(per_env)) : 2;
    if (want && coop && sms > 0 && !slab_mode && !e->aa && e->mrt_K.empty() && e->n_own > 0 && nslots < (1ull << 32)) {
      for (int per_sm = first; per_sm >= 1 && !e->res_blocks; --per_sm) {
        const int ctas = sms * per_sm;
        if (ctas > splbm_dev::kResidentMaxCtas) continue;
        const uint64_t tpc = (e->n_own + ctas - 1) / ctas;
        const uint64_t threads = (tpc * n_tn + 31) / 32 * 32;
        if (splbm_dev::resident_fits(d, e->incompressible != 0, e->f32, static_cast<unsigned>(threads),
                                     static_cast<unsigned>(per_sm)) != cudaSuccess)
          continue;
        e->res_tpc = static_cast<int>(tpc);
        e->res_threads = static_cast<unsigned>(threads);
        e->res_blocks = static_cast<unsigned>((e->n_own + tpc - 1) / tpc);
        e->res_flags = e->alloc<unsigned>(32ull * e->res_blocks);
        CK(cudaMemset(e->res_flags, 0, 32ull * e->res_blocks * sizeof(unsigned)));
      }
      cudaGetLastError();  // a rejected probe leaves no sticky error; clear the last-error slot
    }
  }
}

// GPU-built engines keep the tile cover on the device until a caller needs the host TileMap
// (tile-grid export, fields); then it is downloaded once and the device copies are released.
void host_tm(splbm_dev_engine* e) {
  if (!e->tb.tile_map) return;
  TileMap& tm = e->tm;
  const uint64_t T = tm.n_tiles;
  const uint64_t C = static_cast<uint64_t>(tm.grid_dims[0]) * tm.grid_dims[1] * tm.grid_dims[2];
  tm.tile_map.resize(C);
  tm.origins.resize(T * 3);
  tm.fluid_count.resize(T);
  tm.types.resize(T * tm.n_tn);
  std::vector<uint32_t> cell(T);
  CK(cudaMemcpy(tm.tile_map.data(), e->tb.tile_map, C * 4, cudaMemcpyDeviceToHost));
  if (T) {
    CK(cudaMemcpy(cell.data(), e->tb.cell_of, T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tm.fluid_count.data(), e->tb.fluid_count, T * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tm.types.data(), e->tb.types, T * tm.n_tn, cudaMemcpyDeviceToHost));
  }
  const int* gd = tm.grid_dims;
  const int az = tm.d == 3 ? tm.a : 1;
  for (uint64_t t = 0; t < T; ++t) {
    const uint64_t c = cell[t];
    tm.origins[3 * t] = static_cast<int32_t>(c % gd[0]) * tm.a;
    tm.origins[3 * t + 1] = static_cast<int32_t>((c / gd[0]) % gd[1]) * tm.a;
    tm.origins[3 * t + 2] = static_cast<int32_t>(c / (static_cast<uint64_t>(gd[0]) * gd[1])) * az;
  }
  splbm_dev::free_tile_build(&e->tb);
  e->device_bytes -= e->tb_bytes;
  e->tb_bytes = 0;
}

// A single-copy slab engine in the swapped layout has some of its post-collision values in the
// neighbours' memory (p2p) or in its halo copies: its state is readable after an even step count.
void natural_slab_state(const splbm_dev_engine* e) {
  if (e->aa && e->read == 1 && (e->n_low || e->n_high))
    throw config_error("single-copy slab state is readable after an even number of steps");
}

void check_domain_flag(splbm_dev_engine* e, const char* msg) {
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, e->domain_err, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  if (flag) throw domain_error(msg);
}

void read_failure(splbm_dev_engine* e, int* ok_out, long* failed_out) {
  unsigned long long f = 0;
  CK(cudaMemcpyAsync(&f, e->failed, sizeof(f), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  e->pending_steps = 0;
  if (ok_out) *ok_out = f == ULLONG_MAX ? 1 : 0;
  if (failed_out) *failed_out = f == ULLONG_MAX ? 0 : static_cast<long>(f);
}

}  // namespace

extern "C" {

const char* splbm_last_error(void) { return g_last_error.c_str(); }
const char* splbm_version(void) { return "splbm_b200 0.1 (sm_100a)"; }
size_t splbm_dev_info_size(void) { return sizeof(splbm_dev_info); }

int splbm_dev_create(const splbm_dev_desc* desc, splbm_dev_engine** out) {
  if (!out) return SPLBM_ERR_CONFIG;
  *out = nullptr;
  auto e = std::make_unique<splbm_dev_engine>();
  e->device = desc ? desc->device : 0;
  const int rc = guarded([&] { build(e.get(), desc); });
  if (rc == SPLBM_OK) *out = e.release();
  return rc;
}

void splbm_dev_destroy(splbm_dev_engine* e) { delete e; }

int splbm_dev_get_info(const splbm_dev_engine* e, splbm_dev_info* out) {
  return guarded([&] {
    if (!e || !out) throw config_error("null argument");
    out->n_tiles = e->n_own;
    out->n_tiles_stored = e->n_stored;
    out->n_tn = e->n_tn;
    out->q = e->q;
    out->a = e->a;
    out->d = e->d;
    for (int k = 0; k < 3; ++k) {
      out->grid_dims[k] = e->tm.grid_dims[k];
      out->padded_dims[k] = e->tm.padded_dims[k];
    }
    out->fluid_nodes = e->fluid_nodes;
    out->device_bytes = e->device_bytes;
    out->phi_t = e->n_own ? static_cast<double>(e->fluid_nodes) / (static_cast<double>(e->n_own) * e->n_tn) : 0.0;
    const double cells = static_cast<double>(e->tm.grid_dims[0]) * e->tm.grid_dims[1] * e->tm.grid_dims[2];
    out->ratio_tiles = e->tm.n_tiles ? cells / static_cast<double>(e->tm.n_tiles) : 0.0;
    out->n_tiles_global = e->tm.n_tiles;
    out->resident_ctas = static_cast<int>(e->res_blocks);
    out->resident_threads = static_cast<int>(e->res_threads);
    out->mrt_specialised = e->mrt_jit_ok ? 1 : 0;
  });
}

int splbm_dev_get_tile_grid(const splbm_dev_engine* e, uint32_t* tile_map, int32_t* origins,
                            uint8_t* tile_types, uint32_t* fluid_count, uint32_t* nb) {
  return guarded([&] {
    if (!e) throw config_error("null engine");
    CK(cudaSetDevice(e->device));
    host_tm(const_cast<splbm_dev_engine*>(e));
    const TileMap& tm = e->tm;
    if (tile_map) std::memcpy(tile_map, tm.tile_map.data(), tm.tile_map.size() * 4);
    if (origins) std::memcpy(origins, tm.origins.data(), tm.origins.size() * 4);
    if (tile_types) std::memcpy(tile_types, tm.types.data(), tm.types.size());
    if (fluid_count) std::memcpy(fluid_count, tm.fluid_count.data(), tm.fluid_count.size() * 4);
    if (nb) {
      const auto n = neighbour_table(tm);
      std::memcpy(nb, n.data(), n.size() * 4);
    }
  });
}

int splbm_dev_stored_tiles(const splbm_dev_engine* e, uint64_t* global_ids) {
  return guarded([&] {
    if (!e || !global_ids) throw config_error("null argument");
    for (uint64_t s = 0; s < e->n_stored; ++s) {
      if (s < e->n_low) global_ids[s] = e->g_low0 + s;
      else if (s < e->n_low + e->n_own) global_ids[s] = e->g_own0 + (s - e->n_low);
      else global_ids[s] = e->g_high0 + (s - e->n_low - e->n_own);
    }
  });
}

static int initialize_impl(splbm_dev_engine* e, const double* rho, const double* ux,
                           const double* uy, const double* uz, double rho0, const double* u0) {
  return guarded([&] {
    checked(e);
    const uint64_t total = e->n_stored * e->n_tn;
    CK(cudaMemsetAsync(e->domain_err, 0, sizeof(int), e->stream));
    for (uint64_t node0 = 0; node0 < total; node0 += kChunkNodes) {
      const uint64_t cnt = std::min(kChunkNodes, total - node0);
      splbm_dev::InitArgs ia{};
      ia.pdf0 = e->pdf[0];
      ia.pdf1 = e->pdf[1];  // nullptr in single-copy mode
      ia.node0 = node0;
      ia.count = cnt;
      ia.n_tn = e->n_tn;
      ia.domain_error = e->domain_err;
      if (rho) {
        double* s = e->scratch;
        CK(cudaMemcpyAsync(s, rho + node0, cnt * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(s + cnt, ux + node0, cnt * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(s + 2 * cnt, uy + node0, cnt * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(s + 3 * cnt, uz + node0, cnt * 8, cudaMemcpyHostToDevice, e->stream));
        ia.rho = s;
        ia.ux = s + cnt;
        ia.uy = s + 2 * cnt;
        ia.uz = s + 3 * cnt;
      } else {
        ia.rho0 = rho0;
        ia.u0[0] = u0[0];
        ia.u0[1] = u0[1];
        ia.u0[2] = u0[2];
      }
      CK(splbm_dev::launch_init(e->d, e->incompressible != 0, e->f32, ia, e->stream));
      ++e->launches;
    }
    check_domain_flag(e, "equilibrium requires rho > 0 for the quasi-compressible model");
    e->read = 0;
    e->step_count = 0;  // engine.hpp:350-351
    CK(cudaMemsetAsync(e->step_base, 0, sizeof(long long), e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

int splbm_dev_initialize(splbm_dev_engine* e, const double* rho, const double* ux,
                         const double* uy, const double* uz) {
  if (!rho || !ux || !uy || !uz) {
    set_last_error("null initial field");
    return SPLBM_ERR_CONFIG;
  }
  return initialize_impl(e, rho, ux, uy, uz, 0.0, nullptr);
}

int splbm_dev_initialize_uniform(splbm_dev_engine* e, double rho, const double u[3]) {
  const double zero[3] = {0.0, 0.0, 0.0};
  return initialize_impl(e, nullptr, nullptr, nullptr, nullptr, rho, u ? u : zero);
}

int splbm_dev_step_async(splbm_dev_engine* e, long nsteps) {
  return guarded([&] {
    checked(e);
    if (nsteps < 0) throw config_error("steps must be non-negative");
    if (e->pending_steps == 0) {
      CK(cudaMemsetAsync(e->failed, 0xff, sizeof(unsigned long long), e->stream));
    }
    // instantiate the batch graph (host work) before the timing event, not inside the batch
    if (nsteps >= kGraphSteps && !e->comm && !e->p2p && !e->res_blocks) e->graph_for(e->read);
    CK(cudaEventRecord(e->ev0, e->stream));
    e->enqueue_steps(nsteps);
    CK(cudaEventRecord(e->ev1, e->stream));
    e->batch_timed = true;
    e->pending_steps += nsteps;
  });
}

int splbm_dev_step_part(splbm_dev_engine* e, int part) {
  return guarded([&] {
    checked(e);
    if (part != 1 && part != 2) throw config_error("step part must be 1 (boundary planes) or 2");
    if (part == 1 && e->pending_steps == 0) {
      CK(cudaMemsetAsync(e->failed, 0xff, sizeof(unsigned long long), e->stream));
    }
    e->step_part(part);
    if (part == 2) ++e->pending_steps;
  });
}

int splbm_dev_sync(splbm_dev_engine* e, int* ok_out, long* failed_step_out) {
  return guarded([&] {
    checked(e);
    read_failure(e, ok_out, failed_step_out);
  });
}

int splbm_dev_step(splbm_dev_engine* e, long nsteps, int* ok_out, long* failed_step_out) {
  int rc = splbm_dev_step_async(e, nsteps);
  if (rc != SPLBM_OK) return rc;
  return splbm_dev_sync(e, ok_out, failed_step_out);
}

long splbm_dev_current_step(const splbm_dev_engine* e) { return e ? e->step_count : 0; }
uint64_t splbm_dev_tile_visits(const splbm_dev_engine* e) { return e ? e->visits : 0; }
uint64_t splbm_dev_launch_count(const splbm_dev_engine* e) { return e ? e->launches : 0; }

int splbm_dev_padded_dims(const splbm_dev_engine* e, int out[3]) {
  if (!e || !out) return SPLBM_ERR_CONFIG;
  for (int k = 0; k < 3; ++k) out[k] = e->tm.padded_dims[k];
  return SPLBM_OK;
}

int splbm_dev_fields(splbm_dev_engine* e, double* rho, double* ux, double* uy, double* uz,
                     uint8_t* mask, double* mass_out) {
  return guarded([&] {
    checked(e);
    natural_slab_state(e);
    const int* dims = e->tm.dims;
    const std::size_t n = static_cast<std::size_t>(dims[0]) * dims[1] * dims[2];
    std::vector<double> own_rho;
    std::vector<uint8_t> own_mask;
    if (mass_out && !rho) {
      own_rho.resize(n);
      rho = own_rho.data();
    }
    if (mass_out && !mask) {
      own_mask.resize(n);
      mask = own_mask.data();
    }
    // The FieldData frame (engine.hpp:516-534: zeros, the moments and mask at non-solid nodes) is
    // assembled on the device in raster order, a chunk of tile layers (z in 3D, y in 2D: the
    // slowest axis of the compact tile order, tiling.cpp:113-141) at a time, and copied straight
    // into the caller's arrays. Layers without owned tiles are zeroed on the host.
    const int a = e->a, d = e->d;
    const int* gd = e->tm.grid_dims;
    const int n_layers = d == 3 ? gd[2] : gd[1];
    const uint64_t plane = d == 3 ? static_cast<uint64_t>(dims[0]) * dims[1] : static_cast<uint64_t>(dims[0]);
    const uint64_t layer_nodes = static_cast<uint64_t>(a) * plane;
    if (!e->frame) {
      host_tm(e);
      std::vector<uint32_t> cells(std::max<uint64_t>(e->n_own, 1));
      e->layer_first.assign(n_layers + 1, e->n_own);
      const int az = d == 3 ? a : 1;
      for (uint64_t i = e->n_own; i-- > 0;) {
        const int32_t* o = &e->tm.origins[3 * (e->g_own0 + i)];
        const uint64_t c = static_cast<uint64_t>(o[0] / a) +
                           static_cast<uint64_t>(gd[0]) * (o[1] / a + static_cast<uint64_t>(gd[1]) * (o[2] / az));
        if (c > 0xffffffffull) throw config_error("fields: more than 2^32 tile cells");
        cells[i] = static_cast<uint32_t>(c);
        const int layer = d == 3 ? o[2] / az : o[1] / a;
        e->layer_first[layer] = i;
      }
      for (int L = n_layers; L-- > 0;)  // layers without tiles start where the next layer does
        e->layer_first[L] = std::min(e->layer_first[L], e->layer_first[L + 1]);
      e->cells = e->alloc<uint32_t>(cells.size());
      CK(cudaMemcpy(e->cells, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice));
      constexpr uint64_t kFrameBytes = 256ull << 20;
      const uint64_t layers = std::max<uint64_t>(1, std::min<uint64_t>(n_layers, kFrameBytes / (33 * layer_nodes)));
      e->frame_nodes = std::min<uint64_t>(layers * layer_nodes, n);
      e->frame = e->alloc<uint8_t>(33 * e->frame_nodes);
    }
    const int per_chunk = static_cast<int>(std::max<uint64_t>(1, e->frame_nodes / layer_nodes));
    double* out[4] = {rho, ux, uy, uz};
    CK(cudaMemsetAsync(e->domain_err, 0, sizeof(int), e->stream));
    for (int L0 = 0; L0 < n_layers; L0 += per_chunk) {
      const int L1 = std::min(n_layers, L0 + per_chunk);
      const uint64_t base = L0 * layer_nodes, cnt = std::min<uint64_t>(n, L1 * layer_nodes) - base;
      const uint64_t i0 = e->layer_first[L0], i1 = e->layer_first[L1];
      if (i0 == i1) {  // no owned tiles: a zero slice
        parallel_for(cnt, [&](std::size_t b, std::size_t en) {
          for (double* o : out)
            if (o) std::memset(o + base + b, 0, (en - b) * 8);
          if (mask) std::memset(mask + base + b, 0, en - b);
        }, 1u << 20);
        continue;
      }
      const uint64_t fn = e->frame_nodes;
      double* fr = reinterpret_cast<double*>(e->frame);
      uint8_t* fm = e->frame + 32 * fn;
      for (int c = 0; c < 4; ++c)
        if (out[c]) CK(cudaMemsetAsync(fr + c * fn, 0, cnt * 8, e->stream));
      if (mask) CK(cudaMemsetAsync(fm, 0, cnt, e->stream));
      splbm_dev::FrameArgs fa{};
      fa.pdf = e->cur_pdf();
      fa.info = e->info;
      fa.view = e->view();
      fa.cells = e->cells + i0;
      fa.tile0 = e->n_low + i0;
      fa.n_tiles = i1 - i0;
      fa.n_tn = e->n_tn;
      fa.a = a;
      fa.gx = gd[0];
      fa.gy = gd[1];
      for (int k = 0; k < 3; ++k) fa.dims[k] = dims[k];
      fa.base = base;
      fa.rho = rho ? fr : nullptr;
      fa.ux = ux ? fr + fn : nullptr;
      fa.uy = uy ? fr + 2 * fn : nullptr;
      fa.uz = uz ? fr + 3 * fn : nullptr;
      fa.mask = mask ? fm : nullptr;
      fa.domain_error = e->domain_err;
      CK(splbm_dev::launch_frame(d, e->incompressible != 0, e->f32, fa, e->stream));
      ++e->launches;
      for (int c = 0; c < 4; ++c)
        if (out[c]) CK(cudaMemcpyAsync(out[c] + base, fr + c * fn, cnt * 8, cudaMemcpyDeviceToHost, e->stream));
      if (mask) CK(cudaMemcpyAsync(mask + base, fm, cnt, cudaMemcpyDeviceToHost, e->stream));
    }
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, e->domain_err, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    if (flag) throw domain_error("moments: zero density under the quasi-compressible model");
    if (mass_out) {  // FieldData::total_mass, sequential raster order (fields.hpp:25-31)
      double m = 0.0;
      for (std::size_t i = 0; i < n; ++i)
        if (mask[i]) m += rho[i];
      *mass_out = m;
    }
  });
}

int splbm_dev_reduce(splbm_dev_engine* e, double out[3]) {
  return guarded([&] {
    checked(e);
    natural_slab_state(e);
    const int blocks = 1184;  // 8 x 148 SMs, fixed so the summation order is fixed
    if (!e->reduce_buf) e->reduce_buf = e->alloc<double>(3 * blocks + 3);  // kept: no per-call cudaMalloc
    double* dev = e->reduce_buf;
    splbm_dev::ReduceArgs ra{e->cur_pdf(), e->info, e->view(), e->n_low * e->n_tn,
                             e->n_own * e->n_tn, e->n_tn, dev};
    cudaError_t err = splbm_dev::launch_reduce(e->d, e->incompressible != 0, e->f32, ra, blocks,
                                               dev + 3 * blocks, e->stream);
    e->launches += 2;
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(out, dev + 3 * blocks, 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream);
    if (err == cudaSuccess) err = cudaStreamSynchronize(e->stream);
    CK(err);
  });
}

int splbm_dev_get_pdf(splbm_dev_engine* e, void* f_out) {
  return guarded([&] {
    checked(e);
    natural_slab_state(e);
    const uint64_t tile_bytes = e->tile_stride() * e->es;
    char* out = static_cast<char*>(f_out);
    if (!e->view().swapped) {
      CK(cudaMemcpyAsync(out, e->cur_pdf(), e->n_stored * tile_bytes, cudaMemcpyDeviceToHost,
                         e->stream));
    } else {  // swapped single-copy state: natural layout through the staging buffer, by tiles
      const uint64_t scratch_bytes = 8 * std::max<uint64_t>(4 * std::min<uint64_t>(kChunkNodes, std::max<uint64_t>(e->n_stored * e->n_tn, 1)), e->tile_stride());
      const uint64_t per = std::max<uint64_t>(1, scratch_bytes / tile_bytes);
      for (uint64_t t0 = 0; t0 < e->n_stored; t0 += per) {
        const uint64_t nt = std::min(per, e->n_stored - t0);
        CK(splbm_dev::launch_unswap(e->d, e->f32, e->cur_pdf(), e->info, e->view(), e->n_tn, t0,
                                    nt, e->scratch, e->stream));
        ++e->launches;
        CK(cudaMemcpyAsync(out + t0 * tile_bytes, e->scratch, nt * tile_bytes,
                           cudaMemcpyDeviceToHost, e->stream));
      }
    }
    CK(cudaStreamSynchronize(e->stream));
  });
}

int splbm_dev_set_pdf(splbm_dev_engine* e, const void* f) {
  return guarded([&] {
    checked(e);
    if (e->aa) e->read = 0;  // a natural-layout state
    CK(cudaMemcpyAsync(e->cur_pdf(), f, e->n_stored * e->tile_stride() * e->es,
                       cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  });
}

void* splbm_dev_stream(splbm_dev_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

int splbm_dev_last_batch_ms(splbm_dev_engine* e, float* ms_out) {
  return guarded([&] {
    checked(e);
    if (!e->batch_timed) throw config_error("no timed batch yet");
    CK(cudaEventSynchronize(e->ev1));
    CK(cudaEventElapsedTime(ms_out, e->ev0, e->ev1));
  });
}

int splbm_dev_halo_bytes(const splbm_dev_engine* e, uint64_t* low_bytes, uint64_t* high_bytes) {
  if (!e) return SPLBM_ERR_CONFIG;
  const uint64_t face = static_cast<uint64_t>(e->n_tn / e->a) * e->n_halo_dirs * 8;
  if (low_bytes) *low_bytes = e->send_low_tiles * face;
  if (high_bytes) *high_bytes = e->send_high_tiles * face;
  return SPLBM_OK;
}

int splbm_dev_halo_recv_bytes(const splbm_dev_engine* e, uint64_t* low_bytes, uint64_t* high_bytes) {
  if (!e) return SPLBM_ERR_CONFIG;
  const uint64_t face = static_cast<uint64_t>(e->n_tn / e->a) * e->n_halo_dirs * 8;
  if (low_bytes) *low_bytes = e->n_low * face;
  if (high_bytes) *high_bytes = e->n_high * face;
  return SPLBM_OK;
}

// pack: low_dev <- bottom owned plane, layer 0, directions leaving downwards (axis comp -1);
//       high_dev <- top owned plane, layer a-1, directions leaving upwards (axis comp +1).
int splbm_dev_halo_pack(splbm_dev_engine* e, void* low_dev, void* high_dev) {
  return guarded([&] {
    checked(e);
    e->pack_faces(e->read, static_cast<double*>(low_dev), static_cast<double*>(high_dev));
  });
}

// pack_next: as pack, from the copy the in-flight step is writing (after step part 1).
int splbm_dev_halo_pack_next(splbm_dev_engine* e, void* low_dev, void* high_dev) {
  return guarded([&] {
    checked(e);
    e->pack_faces(1 - e->read, static_cast<double*>(low_dev), static_cast<double*>(high_dev));
  });
}

// unpack: low_dev (the lower neighbour's high face) -> low halo plane, layer a-1, upward dirs;
//         high_dev (the upper neighbour's low face) -> high halo plane, layer 0, downward dirs.
int splbm_dev_halo_unpack(splbm_dev_engine* e, const void* low_dev, const void* high_dev) {
  return guarded([&] {
    checked(e);
    e->unpack_faces(e->read, const_cast<double*>(static_cast<const double*>(low_dev)),
                    const_cast<double*>(static_cast<const double*>(high_dev)));
  });
}

int splbm_dev_halo_pack_back(splbm_dev_engine* e, void* low_dev, void* high_dev) {
  return guarded([&] {
    checked(e);
    e->pack_back(static_cast<double*>(low_dev), static_cast<double*>(high_dev));
  });
}

int splbm_dev_halo_unpack_back(splbm_dev_engine* e, const void* low_dev, const void* high_dev) {
  return guarded([&] {
    checked(e);
    e->unpack_back(const_cast<double*>(static_cast<const double*>(low_dev)),
                   const_cast<double*>(static_cast<const double*>(high_dev)));
  });
}

// IPC blob of a slab engine: what a neighbour needs to store faces into this engine's halos.
struct IpcBlob {
  uint32_t magic, version;
  int32_t pid, device;
  cudaIpcMemHandle_t pdf[2], flags;
  uint64_t raw_pdf[2], raw_flags;  // same-process peers use the pointers directly
  uint64_t n_low, n_own, n_high, send_low_tiles, send_high_tiles, tile_stride;
  uint32_t single_copy;
};
static_assert(sizeof(IpcBlob) <= SPLBM_IPC_BLOB_BYTES, "blob too large");

int splbm_dev_ipc_blob(splbm_dev_engine* e, uint8_t* out) {
  return guarded([&] {
    checked(e);
    if (!out) throw config_error("null argument");
    if (!e->flags) {
      e->flags = e->alloc<unsigned long long>(2);
      CK(cudaMemset(e->flags, 0, 2 * sizeof(unsigned long long)));
    }
    IpcBlob b{};
    b.magic = 0x53504c42u;  // "SPLB"
    b.version = 2;
    b.pid = static_cast<int32_t>(getpid());
    b.device = e->device;
    for (int k = 0; k < 2; ++k) {
      if (!e->pdf[k]) continue;  // single copy: one array
      CK(cudaIpcGetMemHandle(&b.pdf[k], e->pdf[k]));
      b.raw_pdf[k] = reinterpret_cast<uint64_t>(e->pdf[k]);
    }
    b.single_copy = e->aa ? 1u : 0u;
    CK(cudaIpcGetMemHandle(&b.flags, e->flags));
    b.raw_flags = reinterpret_cast<uint64_t>(e->flags);
    b.n_low = e->n_low;
    b.n_own = e->n_own;
    b.n_high = e->n_high;
    b.send_low_tiles = e->send_low_tiles;
    b.send_high_tiles = e->send_high_tiles;
    b.tile_stride = e->tile_stride();
    std::memset(out, 0, SPLBM_IPC_BLOB_BYTES);
    std::memcpy(out, &b, sizeof(b));
  });
}

int splbm_dev_p2p_attach(splbm_dev_engine* e, const uint8_t* lower_blob, const uint8_t* upper_blob) {
  return guarded([&] {
    checked(e);
    if (e->p2p || e->comm) throw config_error("engine already has a halo transport");
    if (e->f32) throw config_error("slab halo exchange is built for the f64 engine");
    if (!e->mrt_K.empty()) throw config_error("peer-store halos are built for the BGK kernels");
    if (!e->flags) throw config_error("call splbm_dev_ipc_blob before attaching");
    if (e->a != 4 && e->a != 2 && !(e->d == 2 && (e->a == 8 || e->a == 16)))
      throw config_error("peer-store halos need a power-of-two tile kernel (a = 2, 4; 2D a <= 16)");
    auto open = [&](const IpcBlob& b, double** pdf, unsigned long long** fl) {
      if (b.magic != 0x53504c42u || b.version != 2 || b.tile_stride != e->tile_stride() ||
          b.single_copy != (e->aa ? 1u : 0u))
        throw config_error("incompatible peer blob");
      if (b.pid == static_cast<int32_t>(getpid())) {
        if (b.device != e->device) {  // one process driving several GPUs: direct peer access
          int can = 0;
          CK(cudaDeviceCanAccessPeer(&can, e->device, b.device));
          if (!can)
            throw Error(SPLBM_ERR_CUDA, "device " + std::to_string(e->device) +
                                            " cannot access peer device " + std::to_string(b.device));
          const cudaError_t pe = cudaDeviceEnablePeerAccess(b.device, 0);
          if (pe == cudaErrorPeerAccessAlreadyEnabled)
            (void)cudaGetLastError();  // enabled by an earlier engine: fine
          else
            CK(pe);
        }
        pdf[0] = reinterpret_cast<double*>(b.raw_pdf[0]);
        pdf[1] = reinterpret_cast<double*>(b.raw_pdf[1]);
        *fl = reinterpret_cast<unsigned long long*>(b.raw_flags);
        return;
      }
      for (int k = 0; k < 2; ++k) {
        if (!b.raw_pdf[k]) {
          pdf[k] = nullptr;
          continue;
        }
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, b.pdf[k], cudaIpcMemLazyEnablePeerAccess));
        e->ipc_opened.push_back(p);
        pdf[k] = static_cast<double*>(p);
      }
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, b.flags, cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p);
      *fl = static_cast<unsigned long long*>(p);
    };
    if (lower_blob) {
      IpcBlob b;
      std::memcpy(&b, lower_blob, sizeof(b));
      if (b.n_high != e->send_low_tiles) throw config_error("lower neighbour's halo does not match my bottom plane");
      open(b, e->peer_pdf_down, &e->peer_flags_down);
      e->peer_down_halo0 = b.n_low + b.n_own;
      e->peer_down_own0 = b.n_low + b.n_own - b.send_high_tiles;
      if (e->aa && b.send_high_tiles != e->n_low)
        throw config_error("lower neighbour's top plane does not match my low halo");
    }
    if (upper_blob) {
      IpcBlob b;
      std::memcpy(&b, upper_blob, sizeof(b));
      if (b.n_low != e->send_high_tiles) throw config_error("upper neighbour's halo does not match my top plane");
      open(b, e->peer_pdf_up, &e->peer_flags_up);
      e->peer_up_own0 = b.n_low;
      if (e->aa && b.send_low_tiles != e->n_high)
        throw config_error("upper neighbour's bottom plane does not match my high halo");
    }
    stream_mem_ops();
    {
      CUdevice cu_dev = 0;
      int can_flush = 0;
      CUresult (*get_dev)(CUdevice*, int) = nullptr;
      CUresult (*get_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
      cudaDriverEntryPointQueryResult q1, q2;
      void* p1 = nullptr;
      void* p2 = nullptr;
      if (cudaGetDriverEntryPoint("cuDeviceGet", &p1, cudaEnableDefault, &q1) == cudaSuccess &&
          cudaGetDriverEntryPoint("cuDeviceGetAttribute", &p2, cudaEnableDefault, &q2) == cudaSuccess &&
          p1 && p2 && q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
        get_dev = reinterpret_cast<decltype(get_dev)>(p1);
        get_attr = reinterpret_cast<decltype(get_attr)>(p2);
        if (get_dev(&cu_dev, e->device) == CUDA_SUCCESS)
          get_attr(&can_flush, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, cu_dev);
      }
      e->wait_flush = can_flush != 0;
      if (const char* v = std::getenv("SPLBM_P2P_WAIT")) {
        if (std::strcmp(v, "kernel") == 0) e->wait_flush = false;
        else if (std::strcmp(v, "flush") == 0) {
          if (!can_flush) throw config_error("SPLBM_P2P_WAIT=flush: device cannot flush remote writes");
          e->wait_flush = true;
        }
      }
    }
    CK(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    e->zero_base = e->alloc<long long>(1);
    CK(cudaMemset(e->zero_base, 0, sizeof(long long)));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&e->ev_int[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&e->ev_bnd[k], cudaEventDisableTiming));
    }
    e->p2p = true;
  });
}

int splbm_comm_unique_id(uint8_t* id_out) {
  return guarded([&] {
    if (!id_out) throw config_error("null argument");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, sizeof(id.internal));
  });
}

int splbm_dev_comm_attach(splbm_dev_engine* e, const uint8_t* id, int world, int rank,
                          int lower_rank, int upper_rank) {
  return guarded([&] {
    checked(e);
    if (e->comm) throw config_error("engine already has a communicator");
    if (e->aa) throw config_error("slab halo exchange needs the two-copy scheme");
    if (e->f32) throw config_error("slab halo exchange is built for the f64 engine");
    if (!id || world < 1 || rank < 0 || rank >= world || lower_rank >= world || upper_rank >= world)
      throw config_error("invalid communicator arguments");
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    const uint64_t face = static_cast<uint64_t>(e->n_tn / e->a) * e->n_halo_dirs;
    e->halo_n[0] = e->send_low_tiles * face;
    e->halo_n[1] = e->send_high_tiles * face;
    e->halo_n[2] = e->n_low * face;
    e->halo_n[3] = e->n_high * face;
    for (int k = 0; k < 4; ++k) e->halo_buf[k] = e->alloc<double>(e->halo_n[k]);
    CK(cudaStreamCreateWithFlags(&e->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&e->ev_packed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->ev_arrived, cudaEventDisableTiming));
    e->lower_rank = lower_rank;
    e->upper_rank = upper_rank;
    nccl_check(nccl().CommInitRank(&e->comm, world, uid, rank), "ncclCommInitRank");
  });
}

int splbm_selftest_divide(uint64_t n, const double* m3, const double* rho, double* out3) {
  return guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(SPLBM_ERR_CUDA, "no CUDA device available");
    double *dm = nullptr, *dr = nullptr, *dout = nullptr;
    const std::size_t nb = std::max<uint64_t>(n, 1) * 8;
    CK(cudaMalloc(&dm, 3 * nb));
    CK(cudaMalloc(&dr, nb));
    CK(cudaMalloc(&dout, 3 * nb));
    cudaError_t err = cudaMemcpy(dm, m3, 3 * n * 8, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(dr, rho, n * 8, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = splbm_dev::launch_divide_selftest(n, dm, dr, dout, nullptr);
    if (err == cudaSuccess) err = cudaMemcpy(out3, dout, 3 * n * 8, cudaMemcpyDeviceToHost);
    cudaFree(dm);
    cudaFree(dr);
    cudaFree(dout);
    CK(err);
  });
}

int splbm_selftest_divide_f32(uint64_t n, const float* m3, const float* rho, float* out3) {
  return guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(SPLBM_ERR_CUDA, "no CUDA device available");
    float *dm = nullptr, *dr = nullptr, *dout = nullptr;
    const std::size_t nb = std::max<uint64_t>(n, 1) * 4;
    CK(cudaMalloc(&dm, 3 * nb));
    CK(cudaMalloc(&dr, nb));
    CK(cudaMalloc(&dout, 3 * nb));
    cudaError_t err = cudaMemcpy(dm, m3, 3 * n * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(dr, rho, n * 4, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = splbm_dev::launch_divide_selftest_f32(n, dm, dr, dout, nullptr);
    if (err == cudaSuccess) err = cudaMemcpy(out3, dout, 3 * n * 4, cudaMemcpyDeviceToHost);
    cudaFree(dm);
    cudaFree(dr);
    cudaFree(dout);
    CK(err);
  });
}

}  // extern "C"
