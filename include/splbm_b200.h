/*
 * splbm_b200 — B200-native (sm_100a) time-step path for the tiled sparse lattice Boltzmann
 * solver of arXiv 1703.08015 (reference: `splbm`, /root/reference/proj).
 *
 * This is the drop-in boundary: a C ABI (plain pointers and sizes, no C++ or torch types)
 * that the reference's `Engine<T>` interface (proj/include/splbm/engine.hpp:67-92) binds to.
 * Each entry point names the reference interface it replaces. All host buffers are copied;
 * the caller keeps ownership. No call throws; every call returns an splbm_status and
 * splbm_last_error() holds the message (thread-local). There is no CPU fallback: without a
 * CUDA device, engine calls fail with SPLBM_ERR_CUDA.
 */
#ifndef SPLBM_B200_H
#define SPLBM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto the reference exception hierarchy (errors.hpp:9-53). */
typedef enum {
  SPLBM_OK = 0,
  SPLBM_ERR_CONFIG = 1,    /* ConfigError   (collision.cpp:90-92, tiling.cpp:87-93) */
  SPLBM_ERR_DOMAIN = 2,    /* DomainError   (lattice.hpp:76-78, 105-108)            */
  SPLBM_ERR_NUMERICAL = 3, /* NumericalError(step) (engine.hpp:634)                 */
  SPLBM_ERR_IO = 4,        /* IoError       (geometry.cpp:358-368)                  */
  SPLBM_ERR_PARSE = 5,     /* ParseError    (geometry.cpp:49-152)                   */
  SPLBM_ERR_CUDA = 6       /* device / driver failure (no reference counterpart)    */
} splbm_status;

#define SPLBM_EMPTY_TILE 0xffffffffu /* kEmptyTile, tiling.hpp:16 */

/* NodeType (geometry.hpp:14): 0 Solid, 1 Fluid, 2 VelocityBC, 3 PressureBC. */
/* Periodicity (tiling.hpp:19-24) as a bit mask: 1 = x, 2 = y, 4 = z. */

const char* splbm_last_error(void);
const char* splbm_version(void);
/* sizeof(splbm_dev_info) as compiled into the library: callers built against another revision of
 * this header compare it with their own sizeof and refuse to run on a mismatch (ABI guard). */
size_t splbm_dev_info_size(void);

/* ---- geometry (geometry.hpp:27-82; input side of the path) -------------------------------- */
typedef enum {
  SPLBM_GEOM_CAVITY2D = 0,  /* generate(Cavity2D)  geometry.cpp:199-224 */
  SPLBM_GEOM_CAVITY3D = 1,  /* generate(Cavity3D)  geometry.cpp:199-224 */
  SPLBM_GEOM_CHANNEL2D = 2, /* generate(Channel2D) geometry.cpp:226-245 */
  SPLBM_GEOM_RAS3D = 3,     /* generate(Ras3D)     geometry.cpp:251-326 */
  SPLBM_GEOM_CHANNEL3D = 4, /* new: 3D duct, walls y,z; V inlet x=0, P outlet x=nx-1 */
  SPLBM_GEOM_VESSEL2D = 5   /* new: seeded binary vessel tree */
} splbm_geometry_kind;

typedef struct {
  int dims[3];           /* nz = 1 for 2D kinds */
  double lid_speed;      /* GenerateParams::lid_speed (0.05) */
  double inlet_speed;    /* GenerateParams::inlet_speed (0.05) */
  double outlet_density; /* GenerateParams::outlet_density (1.0) */
  int sphere_diameter;   /* GenerateParams::sphere_diameter (40) */
  double target_porosity;/* GenerateParams::target_porosity (0.9) */
  uint64_t seed;         /* GenerateParams::seed (0) */
} splbm_generate_params;

/* generate() (geometry.cpp:370-382). types_out: dims[0]*dims[1]*dims[2] bytes, x fastest.
 * Writes the resulting dimension d and BcParams (geometry.hpp:18-21). */
int splbm_generate(int kind, const splbm_generate_params* p, uint8_t* types_out, int* d_out,
                   double bc_velocity_out[3], double* bc_density_out);

/* generate() with the RAS sphere loop on a CUDA device: the same raster, bit for
 * bit, as splbm_generate (the reference's generate_ras, geometry.cpp:251-326; candidate centres
 * from the same mt19937_64 stream, accept/skip/retry decided on the device); the other kinds run
 * the host generator. */
int splbm_generate_device(int kind, const splbm_generate_params* p, int device, uint8_t* types_out,
                          int* d_out, double bc_velocity_out[3], double* bc_density_out);

/* SPLB v1 binary / text formats (geometry.cpp:49-191, 347-368). Two-call protocol for load:
 * call with types_out == NULL to get d/dims, then again with a buffer. */
int splbm_geometry_load(const char* path, int* d_out, int dims_out[3], uint8_t* types_out,
                        double bc_velocity_out[3], double* bc_density_out);
int splbm_geometry_save(const char* path, int binary, int d, const int dims[3],
                        const uint8_t* types, const double bc_velocity[3], double bc_density);

/* ---- tile map (tiling.cpp:85-141, tiling.hpp:93-102, engine.hpp:446-463) --------------------- */
/* grid/padded dims of the uniform a^d cover (tiling.cpp:99-108). */
int splbm_tile_dims(int d, const int dims[3], int a, int grid_dims_out[3], int padded_dims_out[3]);
/* Number of non-empty tiles (fluid_count > 0) — sizes the outputs of splbm_build_tile_map. */
int splbm_count_tiles(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                      uint64_t* n_tiles_out);
/* The tile cover, bit-exact with build_tile_grid: tile_map[C] (compact index in cz->cy->cx
 * order, SPLBM_EMPTY_TILE for dropped cells), origins[T*3], tile_types[T*n_tn] (x-fastest local,
 * padding Solid), fluid_count[T], and (optional, may be NULL) the 27-neighbour table nb[T*27]
 * with nb[t*27 + (dx+1)+3((dy+1)+3(dz+1))] = tile_at(cx+dx, cy+dy, cz+dz). */
int splbm_build_tile_map(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                         uint32_t* tile_map, int32_t* origins, uint8_t* tile_types,
                         uint32_t* fluid_count, uint32_t* nb);
/* Non-empty tiles per tile plane along the last axis (z in 3D, y in 2D): the prefix sums give the
 * contiguous compact-index range of every z-slab, used to balance slabs by tiles. */
int splbm_plane_tile_counts(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                            uint64_t* counts_out);

/* Slab layout of the multi-GPU mode for the owned tile planes [z0, z1): stored tiles are
 * [low halo plane zl][owned][high halo plane zh] (zl/zh = -1 when absent). Optional outputs (may be
 * NULL): the local 27-neighbour table (stored*27; tiles outside the stored set -> EMPTY) and the
 * local tile node types (stored*n_tn; bits 0-1 NodeType, bit 2 bc_degenerate). This is exactly the
 * table set splbm_dev_create builds for a slab engine. */
typedef struct {
  int axis, z0, z1, zl, zh;
  uint64_t n_low, n_own, n_high;
  uint64_t g_low0, g_own0, g_high0;
  uint64_t send_low_tiles, send_high_tiles;
} splbm_slab_layout_t;
int splbm_slab_layout(const uint8_t* types, int d, const int dims[3], int a, int periodic, int z0,
                      int z1, splbm_slab_layout_t* out, uint32_t* nb_local, uint8_t* types_local);

/* degenerate_bc_mask (engine.hpp:110-140) over the raster. */
int splbm_degenerate_bc_mask(const uint8_t* types, int d, const int dims[3], int periodic,
                             uint8_t* mask_out);

/* ---- device engine: TileEngineT2C on one B200 (engine.hpp:311-551) --------------------------- */
typedef struct splbm_dev_engine splbm_dev_engine;

typedef struct {
  /* Geometry (geometry.hpp:27-51): raster copied at create; tile map built on the host */
  int d;
  int dims[3];
  const uint8_t* types;
  double bc_velocity[3];
  double bc_density;
  /* SimConfig / FluidModel (engine.hpp:562-576, lattice.hpp:53-63) */
  int tile;           /* tile edge a >= 2; 0 selects 16 (2D) / 4 (3D) like tile_edge() */
  double tau;         /* > 0.5 (collision.cpp:90) */
  int incompressible; /* Compressibility::Incompressible if nonzero */
  int periodic;       /* bit mask */
  int device;         /* CUDA device ordinal */
  /* z-slab of the tile planes this engine owns, [slab_z0, slab_z1) in tile cells; both 0 = all.
   * Multi-GPU slab mode; the engine then stores its own planes plus one halo plane
   * on each side and exchanges face PDFs through splbm_dev_halo_* each step. */
  int slab_z0, slab_z1;
  /* CollisionKind (lattice.hpp:54): 0 BGK, 1 MRT with K = M^-1 S M (collision.cpp:86-113);
   * mrt_rates = q relaxation rates or NULL for default_mrt_rates (collision.cpp:76-84). */
  int collision;
  const double* mrt_rates;
  /* Propagation storage (no reference counterpart): 0 = two PDF copies swapped per
   * step (the reference T2C scheme, engine.hpp:354-369); 1 = one copy updated in place with the
   * AA access pattern (half the HBM, bit-identical results; power-of-two tiles, no slab). */
  int single_copy;
  /* Real type of the engine: 0 = TileEngineT2C<double>; 1 = TileEngineT2C<float> (PDFs and every
   * node operation in float, the reference's `precision=f32`, tools/splbm.cpp:278; no slab). */
  int single_precision;
} splbm_dev_desc;

typedef struct {
  uint64_t n_tiles;        /* non-empty tiles owned (T) */
  uint64_t n_tiles_stored; /* owned + halo tiles */
  int n_tn, q, a, d;
  int grid_dims[3];
  int padded_dims[3];
  uint64_t fluid_nodes;    /* non-solid nodes owned (N_f, engine.hpp:621) */
  uint64_t device_bytes;   /* HBM held by the engine */
  double phi_t;            /* tile porosity (tiling.cpp:223-225) */
  double ratio_tiles;      /* cells / non-empty tiles (tiling.cpp:227) */
  uint64_t n_tiles_global; /* non-empty tiles of the whole tile map */
  /* Step path: 0 = one step-kernel launch per step (CUDA-graph batches); > 0 = the number of CTAs
   * of the resident multi-step kernel (small whole-domain engines: a batch of steps inside one
   * cooperative grid, a grid barrier between steps; SPLBM_RESIDENT=0 disables it). */
  int resident_ctas;
  int resident_threads;
  /* 1 when the MRT step runs the kernel specialised for this engine's operator (see
   * splbm_mrt_specialise); 0 for BGK, single copy, non-power-of-two tiles or SPLBM_MRT_JIT=0 */
  int mrt_specialised;
} splbm_dev_info;

/* TileEngineT2C(g, a, model, periodic) ctor (engine.hpp:314-334): validates like the reference
 * (tau > 0.5, a >= 2, periodic extents divisible by a), builds the tile map, the per-node
 * gather masks and allocates both PDF copies in HBM. */
int splbm_dev_create(const splbm_dev_desc* desc, splbm_dev_engine** out);
void splbm_dev_destroy(splbm_dev_engine* e);
int splbm_dev_get_info(const splbm_dev_engine* e, splbm_dev_info* out);
/* The engine's (global) tile grid, same arrays as splbm_build_tile_map; any pointer may be NULL. */
int splbm_dev_get_tile_grid(const splbm_dev_engine* e, uint32_t* tile_map, int32_t* origins,
                            uint8_t* tile_types, uint32_t* fluid_count, uint32_t* nb);
/* Global compact index of every stored tile (n_tiles_stored entries; owned tiles in the middle,
 * halo planes first/last in slab mode). Node coordinates for splbm_dev_initialize follow from
 * origins[global] + (p % a, (p / a) % a, p / a^2) (engine.hpp:401-407). */
int splbm_dev_stored_tiles(const splbm_dev_engine* e, uint64_t* global_ids);

/* Engine::initialize(NodeInit) (engine.hpp:336-352): rho/ux/uy/uz are NodeInit evaluated at
 * node_coords(tile, p) for every stored tile node (T*n_tn each, tile-major), equilibrium computed
 * on the device into both copies. initialize_uniform (engine.hpp:72-75) needs no host arrays. */
int splbm_dev_initialize(splbm_dev_engine* e, const double* rho, const double* ux,
                         const double* uy, const double* uz);
int splbm_dev_initialize_uniform(splbm_dev_engine* e, double rho, const double u[3]);

/* Engine::step() (engine.hpp:354-369) nsteps times. *ok_out = 0 if a non-finite moment
 * appeared; *failed_step_out = the first such step number (current_step() based, 1-based),
 * like run_simulation's NumericalError(step) (engine.hpp:634). Blocks until done. */
int splbm_dev_step(splbm_dev_engine* e, long nsteps, int* ok_out, long* failed_step_out);
/* Non-blocking variant: enqueue nsteps on the engine stream; the ok flag is read later by
 * splbm_dev_sync. Used to time batches without a per-step host round trip. */
int splbm_dev_step_async(splbm_dev_engine* e, long nsteps);
int splbm_dev_sync(splbm_dev_engine* e, int* ok_out, long* failed_step_out);

long splbm_dev_current_step(const splbm_dev_engine* e);    /* Engine::current_step()  */
uint64_t splbm_dev_tile_visits(const splbm_dev_engine* e); /* Engine::tile_visits()   */
int splbm_dev_padded_dims(const splbm_dev_engine* e, int out[3]); /* padded_dims()   */

/* Engine::fields() (engine.hpp:371-390): (rho, u) of the current post-collision copy scattered
 * to the unpadded raster (x fastest), zeros and mask 0 at solid nodes; any output may be NULL.
 * *mass_out (may be NULL) = FieldData::total_mass() in its sequential raster order. */
int splbm_dev_fields(splbm_dev_engine* e, double* rho, double* ux, double* uy, double* uz,
                     uint8_t* mask, double* mass_out);
/* Device-side reduction without a raster download: out[0] mass (fixed-order tree sum),
 * out[1] max |u|, out[2] number of non-finite nodes. */
int splbm_dev_reduce(splbm_dev_engine* e, double out[3]);

/* Raw PDF copies for parity dumps: slot (t*q+i)*n_tn+p (engine.hpp:397-399), current copy, in the
 * engine's real type (double, or float for single_precision engines); n_tiles_stored*q*n_tn slots. */
int splbm_dev_get_pdf(splbm_dev_engine* e, void* f_out);
int splbm_dev_set_pdf(splbm_dev_engine* e, const void* f);

/* Streams and timing. The engine launches on its own stream (cudaStream_t as void*). */
void* splbm_dev_stream(splbm_dev_engine* e);
/* Device time of the last splbm_dev_step/step_async batch's step kernels, from CUDA events
 * recorded on the engine stream around the batch (ms). Valid after sync. */
int splbm_dev_last_batch_ms(splbm_dev_engine* e, float* ms_out);
/* Kernel launches issued so far by this engine (all kinds). */
uint64_t splbm_dev_launch_count(const splbm_dev_engine* e);

/* ---- multi-GPU slab mode (no reference counterpart) ------------------------------ */
/* Face halo PDFs of the owned slab along the last axis (z in 3D, y in 2D). pack writes, from the
 * current copy, the bottom owned plane's layer 0 for the directions leaving downwards (low) and
 * the top plane's layer a-1 for the directions leaving upwards (high), sizes from
 * splbm_dev_halo_bytes. unpack stores what the lower neighbour packed as `high` into the low halo
 * plane and what the upper neighbour packed as `low` into the high halo plane (sizes from
 * splbm_dev_halo_recv_bytes). All buffers are device pointers; work is on the engine stream. */
int splbm_dev_halo_bytes(const splbm_dev_engine* e, uint64_t* low_bytes, uint64_t* high_bytes);
int splbm_dev_halo_recv_bytes(const splbm_dev_engine* e, uint64_t* low_bytes, uint64_t* high_bytes);
int splbm_dev_halo_pack(splbm_dev_engine* e, void* low_dev, void* high_dev);
/* Overlapped slab step: part 1 steps the bottom and top owned tile planes into the next copy,
 * splbm_dev_halo_pack_next packs their faces from that copy (so the exchange can start), part 2
 * steps the interior planes while the faces are in flight, then swaps the copies and counts the
 * step. part 1 + part 2 == one splbm_dev_step_async(e, 1). Unpack after part 2. */
int splbm_dev_step_part(splbm_dev_engine* e, int part);
int splbm_dev_halo_pack_next(splbm_dev_engine* e, void* low_dev, void* high_dev);
int splbm_dev_halo_unpack(splbm_dev_engine* e, const void* low_dev, const void* high_dev);
/* Single-copy (single_copy = 1) slab engines. Before a step from the natural layout (current_step
 * even) the faces go forward as above (pack / unpack). After that step the halo slots its scatter
 * wrote go back to their owners: pack_back writes the low halo plane's layer a-1, upward dirs
 * (low, to the lower neighbour; size = recv low bytes) and the high halo plane's layer 0, downward
 * dirs (high, to the upper neighbour); unpack_back stores what the lower neighbour sent as `high`
 * into my bottom plane's layer 0 and what the upper neighbour sent as `low` into my top plane's
 * layer a-1 — only the slots whose downstream node is non-solid (the others belong to this node's
 * own bounce-back). Steps from the swapped layout need no exchange. fields/get_pdf/reduce of a
 * slab engine need the natural layout (an even step count). */
int splbm_dev_halo_pack_back(splbm_dev_engine* e, void* low_dev, void* high_dev);
int splbm_dev_halo_unpack_back(splbm_dev_engine* e, const void* low_dev, const void* high_dev);

/* Native exchange (no per-step host work beyond enqueueing): rank 0 creates an NCCL unique id
 * (128 bytes) and every rank passes it to splbm_dev_comm_attach with its lower/upper slab
 * neighbour (-1 at a non-periodic edge). From then on every splbm_dev_step[_async] step runs
 * boundary planes -> pack -> NCCL send/recv on a side stream -> interior planes -> unpack. */
int splbm_comm_unique_id(uint8_t* id_out);
int splbm_dev_comm_attach(splbm_dev_engine* e, const uint8_t* id, int world, int rank,
                          int lower_rank, int upper_rank);

/* Fused NVLink exchange: the boundary-plane step kernel stores its face values straight into the
 * neighbours' halo tiles (peer memory over NVLink; CUDA IPC across processes), ordered by 64-bit
 * flags with GPU-side stream waits/writes — no pack, no unpack, no host synchronisation. Every rank
 * exports its blob (SPLBM_IPC_BLOB_BYTES bytes), the blobs reach the neighbours out of band, then
 * each rank attaches its lower/upper neighbour's blob (NULL at a non-periodic edge). All ranks
 * must initialize before any rank steps. Single-copy engines: the boundary planes' steps from the
 * natural layout read and write the halo nodes' slots in place in the neighbours' owned tiles
 * (each slot has exactly one reader/writer), so no halo copy is involved at all. */
#define SPLBM_IPC_BLOB_BYTES 512
int splbm_dev_ipc_blob(splbm_dev_engine* e, uint8_t* blob_out);
int splbm_dev_p2p_attach(splbm_dev_engine* e, const uint8_t* lower_blob, const uint8_t* upper_blob);

/* The MRT operator matrix the device applies (q x q row-major), bit-identical to the reference's
 * CollisionOperator<double> (collision.cpp:86-113). */
int splbm_mrt_kernel(int d, double tau, const double* rates, double* K_out);
/* Runtime specialisation of the MRT step (no reference counterpart): engines with collision = MRT
 * on power-of-two tiles step with the power-of-two kernel compiled at creation through NVRTC for
 * their operator K — K's constants folded in, each product K_ij * delta_j computed once per
 * distinct value in column j, every row summed in the reference's order (bit-identical; D3Q19,
 * default rates, tau 0.8: 139 instead of 361 products per node). This entry point reports the
 * product count and, when `tile` > 0, compiles the kernel for that tile edge (NVRTC only, no
 * device needed); an NVRTC failure returns SPLBM_ERR_CUDA with the log in splbm_last_error(). */
int splbm_mrt_specialise(int d, int incompressible, int single_precision, double tau,
                         const double* rates, int tile, int* products_out);

/* ---- self-test ------------------------------------------------------------------------------- */
/* Runs the step kernel's velocity division u_k = m_k / rho (collision.hpp:48) on the device for n
 * (m0, m1, m2, rho) tuples; every quotient must equal IEEE division bit for bit. */
int splbm_selftest_divide(uint64_t n, const double* m3, const double* rho, double* out3);
/* The same for the f32 engine (TileEngineT2C<float>): IEEE binary32 division, bit for bit. */
int splbm_selftest_divide_f32(uint64_t n, const float* m3, const float* rho, float* out3);

#ifdef __cplusplus
}
#endif
#endif /* SPLBM_B200_H */
