/*
 * ts_b200.h -- C ABI of the B200-native LidarScout heightmap hot path.
 *
 * One shared library (paper_2509_20198_b200/libts_b200.so), plain C types,
 * caller-owned device buffers, an explicit cudaStream_t (passed as void*)
 * on every compute entry point.  Nothing here blocks the host except the
 * calls documented as "synchronous" (they size outputs).  Every function is
 * reentrant; the only library-owned state is the opaque weight handle.
 *
 * Each entry point replaces a reference function of the Python package
 * `terrascout` (/root/reference/pkg/src/terrascout); the replaced
 * file:line is cited above each declaration.  INTEGRATION.md shows the
 * ctypes binding the reference would add.
 */
#ifndef TS_B200_H
#define TS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped onto terrascout.errors, errors.py:4-57) ---- */
enum ts_status {
  TS_OK = 0,
  TS_E_EMPTY_PATCH = 1,        /* EmptyPatch        */
  TS_E_EMPTY_SET = 2,          /* EmptySet          */
  TS_E_SHAPE = 3,              /* ShapeMismatch     */
  TS_E_BAD_MAGIC = 4,          /* BadMagic          */
  TS_E_VERSION = 5,            /* UnsupportedVersion*/
  TS_E_CORRUPT_TABLE = 6,      /* CorruptChunkTable */
  TS_E_OOB = 7,                /* OutOfBoundsRead   */
  TS_E_UNSUPPORTED_FORMAT = 8, /* UnsupportedFormat */
  TS_E_CUDA = 9,               /* CUDA runtime error */
  TS_E_DESYNC = 10,            /* DecoderDesync     */
  TS_E_INVALID = 11            /* bad argument      */
};

/* Per-tile metadata parsed on the host from the LAS header
 * (lasio/header.py:109-183 / reader.py:49-73 TileMeta). */
typedef struct ts_tile_desc {
  int64_t file_offset;       /* start of this tile's file image in d_bytes */
  int64_t file_size;         /* bytes of the image                          */
  int64_t point_data_offset; /* LAS point_data_offset                       */
  int64_t point_count;       /* header point count                          */
  int64_t las_stride;        /* LAS (uncompressed) chunk stride (reader.py:212) */
  uint32_t chunk_size;       /* LASzip chunk size, 0xFFFFFFFF = variable    */
  int32_t format;            /* point record format (0..3 supported)        */
  int32_t record_length;     /* header point_record_length                  */
  int32_t compressed;        /* 1 = LAZ (chunk table), 0 = LAS              */
  double scale[3];
  double offset[3];
  /* Sparse images (the file is not uploaded whole): the image in d_bytes
   * holds file bytes [image_base, image_base + image size); 0 = the whole
   * file.  table_pos >= 0: the chunk-table position (the host read the
   * 8-byte pointer, reader.py:146-157); < -1 (TS_TABLE_POS_IN_IMAGE): read
   * the pointer from the image.  file_size is then the real file size.   */
  int64_t image_base;
  int64_t table_pos;
} ts_tile_desc;
#define TS_TABLE_POS_IN_IMAGE (-2)

/* Patch key: centre of a 640 m patch (patches.py:33-53). */
typedef struct ts_patch_key {
  double cx, cy;
} ts_patch_key;

/* ---- library ---- */
const char* ts_version(void);
int ts_device_count(void);
/* Kernels launched by this library since load (launch accounting). */
uint64_t ts_launch_count(void);
/* Bytes of record_dtype(fmt) (lasio/records.py:43-59) for fmt 0..3. */
int ts_record_size(int format);

/* ---- (1) chunk-first-point extraction --------------------------------
 * Replaces read_chunk_table (reader.py:132-209) and read_chunk_points
 * (reader.py:251-283) for a batch of tiles resident in device memory.
 *
 * Step 1: per-tile chunk count (LAZ: u32 at table+4; LAS:
 *         ceil(point_count / las_stride)).  d_n_chunks[n_tiles].          */
int ts_chunk_counts(const uint8_t* d_bytes, const ts_tile_desc* d_tiles,
                    int n_tiles, int64_t* d_n_chunks, int32_t* d_status,
                    void* stream);
/* Step 2: decode every chunk table (LASzip arithmetic-coded
 * IntegerCompressor, codec.py:173-484) into absolute byte offsets and
 * point counts.  d_chunk_base[n_tiles+1] is the exclusive prefix sum of
 * the counts.  d_scratch must hold ts_chunk_decode_scratch(n_tiles) bytes. */
size_t ts_chunk_decode_scratch(int n_tiles);
int ts_chunk_decode(const uint8_t* d_bytes, const ts_tile_desc* d_tiles,
                    int n_tiles, const int64_t* d_chunk_base,
                    int64_t* d_chunk_offset, int64_t* d_chunk_points,
                    int64_t* d_chunk_end, int32_t* d_status, void* d_scratch,
                    void* stream);
/* Step 3: gather + decode the uncompressed first record of every chunk
 * (reader.py:239-283) with 16-byte vector loads; fuse positions()
 * (records.py:62-67, fp64 x*s+o, no FMA) and colors() (records.py:70-86,
 * per-tile 8/16-bit divisor).  Outputs (any may be NULL):
 *   d_records  packed record_dtype(fmt) rows (all tiles must share fmt),
 *   d_xyz      (n,3) float64,  d_rgb (n,3) float32 (colour formats),
 *   d_cell     (n,2) int64 floor(x/640), floor(y/640) (patches.py:119-120). */
int ts_extract_chunk_points(const uint8_t* d_bytes,
                            const ts_tile_desc* d_tiles, int n_tiles,
                            const int64_t* d_chunk_base,
                            const int64_t* d_chunk_offset,
                            uint8_t* d_records, double* d_xyz, float* d_rgb,
                            int64_t* d_cell, int32_t* d_status,
                            void* stream);
/* Full chunk decode (reader.py:286-364 decode_chunk / load_tile_fullres,
 * items.py:108-606 POINT10 / GPSTIME11 / RGB12 v2, codec.py:173-484): every
 * record of every chunk of the tiles in d_bytes, bit-exact, one GPU thread
 * per chunk.  Chunk tables from ts_chunk_counts / ts_chunk_decode (offsets,
 * point counts, d_chunk_end); d_point_base[n_chunks + 1] = exclusive scan
 * of the chunk point counts: chunk c's records land at d_records +
 * d_point_base[c] * record size (all tiles must share the format).
 * d_status[n_chunks]: TS_E_DESYNC (stream ran past the chunk), TS_E_OOB,
 * TS_E_UNSUPPORTED_FORMAT (LAS tiles: read the records directly),
 * TS_E_INVALID (more adaptive models than the per-chunk arena holds).
 * d_scratch: ts_lazdec_scratch(n_chunks) bytes.                          */
size_t ts_lazdec_scratch(int64_t n_chunks);
int ts_lazdec(const uint8_t* d_bytes, const ts_tile_desc* d_tiles, int n_tiles,
              const int64_t* d_chunk_base, const int64_t* d_chunk_offset,
              const int64_t* d_chunk_points, const int64_t* d_chunk_end,
              const int64_t* d_point_base, int64_t n_chunks, uint8_t* d_records,
              int32_t* d_status, void* d_scratch, void* stream);
/* positions()/colors() for records already in device memory
 * (records.py:62-86).  Records are rows of record_stride bytes with x,y,z
 * int32 at bytes 0,4,8 and red,green,blue uint16 at rgb_offset.
 * d_scratch: 1 int32 of device scratch (the per-batch max reduction).   */
int ts_positions(const uint8_t* d_records, int64_t n, int record_stride,
                 const double scale[3], const double offset[3],
                 double* d_xyz, void* stream);
int ts_colors(const uint8_t* d_records, int64_t n, int record_stride,
              int rgb_offset, float* d_rgb, int32_t* d_scratch,
              void* stream);

/* ---- (2) sparse-to-grid rasterisation -------------------------------- */
/* ChunkPointIndex (patches.py:99-160): stable cell order of the points.
 * Cells are dense over [ci0, ci0+nci) x [cj0, cj0+ncj); d_cell_start /
 * d_cell_end have nci*ncj entries (index ci-major like lexsort((cj,ci))).
 * d_order[n] receives point ids sorted by (cell, id).  Synchronous only in
 * that it allocates its own temporary sort storage on the stream.        */
int ts_index_build(const int64_t* d_cell, int64_t n, int64_t ci0,
                   int64_t cj0, int64_t nci, int64_t ncj, int32_t* d_order,
                   int32_t* d_cell_start, int32_t* d_cell_end, void* stream);
/* floor(x/640), floor(y/640) per point (patches.py:119-120), (n,2) int64,
 * for points that did not come through ts_extract_chunk_points.          */
int ts_cell_keys(const double* d_xyz, int64_t n, int64_t* d_cell,
                 void* stream);
/* gather_and_normalize (patches.py:163-177), pass 1: points per patch in
 * the padded square (radius 480 m) -> d_counts[n_patches].               */
int ts_gather_count(const double* d_xyz, const int32_t* d_order,
                    const int32_t* d_cell_start, const int32_t* d_cell_end,
                    int64_t ci0, int64_t cj0, int64_t nci, int64_t ncj,
                    const ts_patch_key* d_keys, int n_patches, double radius,
                    int32_t* d_counts, void* stream);
/* pass 2: ordered gather into CSR slots d_pts_off[n_patches+1] (exclusive
 * scan of counts): xy (2N) and h (N) float64 in patch space, rgb (3N)
 * float32 (if d_rgb), provisional c_z per patch; d_xyz_out (nullable)
 * receives the raw gathered xyz (ChunkPointIndex.query_square,
 * patches.py:131-153; radius != 480 only makes sense with it).  Empty
 * patch -> d_status[p] = TS_E_EMPTY_PATCH.                               */
int ts_gather_fill(const double* d_xyz, const float* d_rgb,
                   const int32_t* d_order, const int32_t* d_cell_start,
                   const int32_t* d_cell_end, int64_t ci0, int64_t cj0,
                   int64_t nci, int64_t ncj, const ts_patch_key* d_keys,
                   int n_patches, double radius, const int64_t* d_pts_off,
                   double* d_xy, double* d_h, float* d_prgb, double* d_cz,
                   double* d_xyz_out, int32_t* d_status, void* stream);
/* nearest_neighbor_query / _nn_assign (patches.py:180-205): exact d^2
 * argmin per query, ties to the lowest index.  n == 0 -> TS_E_EMPTY_SET. */
int ts_nearest(const double* d_xy, int64_t n, const double* d_q, int64_t nq,
               int64_t* d_idx, void* stream);
/* Delaunay triangulation of each patch's points + the 4 padding corners
 * (replaces scipy Delaunay/Qhull at patches.py:316-326).  Exact
 * orientation/incircle predicates; vertex ids 0..N-1 real, N..N+3 the
 * corners (-1,-1),(1,-1),(-1,1),(1,1).  Triangle slot p starts at
 * 2*pts_off[p] + 8*p; capacity 2N+8; d_ntri[p] gets the count.  CCW.
 * Any patch size and insertion order: patches of <= 384 points run in
 * shared memory and restart in global memory if a cavity outgrows it.
 * d_scratch: ts_triangulate_scratch(total points, patches) bytes (the
 * global-memory meshes, circumcircle caches and cavities).                */
size_t ts_triangulate_scratch(int64_t total_points, int n_patches);
int ts_triangulate(const double* d_xy, const int64_t* d_pts_off,
                   int n_patches, int32_t* d_tri, int32_t* d_ntri,
                   int32_t* d_status, void* d_scratch, void* stream);
/* Algorithm 1 rasterisation (patches.py:290-405) given triangles:
 * exact-d^2 NN (lowest index wins), lowest-id face map with the _TriGeom
 * 1e-9 barycentric test, padding-triangle blanking, barycentric hm/rgb,
 * optional re-centring on cell [48,48] (recenter!=0), float32 outputs.
 * Any output pointer may be NULL:
 *   d_cnn_in  B x 96 x 96 x 8 float32 NHWC (hm_nn, hm_lin, rgb_nn, rgb_lin)
 *   d_hm_nn, d_hm_lin  B x 96 x 96;  d_rgb_nn, d_rgb_lin B x 96 x 96 x 3
 *   d_face B x 96 x 96 int32;  d_cz_out[B] float64.                        */
int ts_raster(const double* d_xy, const double* d_h, const float* d_prgb,
              const int64_t* d_pts_off, const int32_t* d_tri,
              const int64_t* d_tri_off, const int32_t* d_ntri,
              const double* d_cz_in, int n_patches, int recenter,
              float* d_cnn_in, float* d_hm_nn, float* d_hm_lin,
              float* d_rgb_nn, float* d_rgb_lin, int32_t* d_face,
              double* d_cz_out, int32_t* d_status, void* stream);

/* ---- (3) CNN refine ----------------------------------------------------
 * Weight bundle from LSWB bytes (refiner.py:258-311 format, descriptor
 * text validated like ArchDescriptor.from_text/validate :92-170).        */
typedef struct ts_weights ts_weights;
int ts_weights_create(const uint8_t* lswb, size_t n_bytes, int precision,
                      ts_weights** out);
int ts_weights_destroy(ts_weights* w);
int ts_weights_is_identity(const ts_weights* w);
/* Bytes of device workspace ts_refine needs for a batch of B tiles. */
size_t ts_refine_workspace(const ts_weights* w, int batch);
/* refine_batch numerics (refiner.py:475-528) on a device batch:
 * d_in  B x 96 x 96 x 8 float32 NHWC (ts_raster's d_cnn_in),
 * d_out B x 64 x 64 x 4 float32 (channel 0 = heights_rel in metres,
 *       1..3 = rgb clamped to [0,1]),
 * d_nonfinite[B] = 1 when the network produced NaN/Inf in the crop; in
 * that case d_out holds the interpolated fallback (crop(hm_lin)*480 and
 * the UNclamped rgb_lin crop), exactly like the reference.               */
int ts_refine(const ts_weights* w, const float* d_in, int batch,
              float* d_out, uint8_t* d_nonfinite, void* d_workspace,
              void* stream);
/* conv2d (refiner.py:330-388): NCHW float32 cross-correlation + bias.
 * precision: 0 CUDA-core fp32, 1 tcgen05 3xTF32, 2 tcgen05 bf16 (shapes
 * the tensor-core kernel cannot take run on the fp32 kernel).            */
int ts_conv2d(const float* d_x, int batch, int c_in, int h, int w,
              const float* d_weight, int c_out, int k, const float* d_bias,
              int stride, int padding, int precision, float* d_y,
              void* stream);

/* ---- (4) full-resolution texel update ---------------------------------
 * bake_fullres (engine.py:416-456) for P patches at once.  Points (M,3)
 * float64 + optional (M,3) float32 rgb.  Texel assignment is the
 * reference predicate floor((x-(cx-320))/10) in IEEE fp64 for every key
 * whose window may hold the point (bit-exact).  Keys are looked up through
 * a host-built CSR grid of cell size 640 m anchored at (gx0, gy0):
 *   d_cell_keys_off[gnx*gny+1], d_cell_keys[...] (key ids per cell);
 *   d_cell_inner[gnx*gny] (nullable): the first d_cell_inner[c] ids of
 *   cell c are the only keys whose window [cx-320, cx+320] (+-1e-6 m)
 *   meets the open square 1 cm inside the cell; points >= 2 cm inside
 *   their cell test only those.
 * prior: heights_rel float32 P x 64 x 64 with base c_z per patch (f64);
 * prior rgb P x 64 x 64 x 3 (NULL = colourless base).  Outputs heights_rel
 * against key_cz, rgb.  d_accum: ts_bake_workspace(P) bytes of scratch.   */
size_t ts_bake_workspace(int n_patches);
int ts_bake(const double* d_xyz, const float* d_rgb, int64_t m,
            const ts_patch_key* d_keys, int n_patches,
            const int32_t* d_cell_keys_off, const int32_t* d_cell_keys,
            const int32_t* d_cell_inner, double gx0, double gy0, int gnx, int gny,
            const float* d_prior_h, const double* d_base_cz,
            const double* d_key_cz, const float* d_prior_rgb,
            float* d_out_h, float* d_out_rgb, void* d_accum, void* stream);

/* Points in any order -> grouped by 640 m cell of the same key grid (a
 * two-pass counting sort: cell rows, then cells), so ts_bake's shared-memory
 * hot-patch accumulation applies
 * to shuffled input too (bake_fullres accepts any point order,
 * engine.py:416-456).  Points outside the grid are placed last.  Order
 * within a cell is unspecified; ts_bake's fixed-point sums do not depend on
 * it.  Grids up to 16,383 cells; m < 2^32.  d_rgb / d_rgb_out both NULL or
 * both set.  d_scratch: ts_bake_bin_scratch(m, gnx, gny) bytes (0: grid
 * too large, call ts_bake on the unsorted points).                        */
size_t ts_bake_bin_scratch(int64_t m, int gnx, int gny);
int ts_bake_bin(const double* d_xyz, const float* d_rgb, int64_t m, double gx0,
                double gy0, int gnx, int gny, double* d_xyz_out, float* d_rgb_out,
                void* d_scratch, void* stream);

/* ---- WireHeightmap records (server.py:126-142 wire_heightmap,
 *      docs/wire.md "WireHeightmap") -------------------------------------
 * Per patch p, back to back at d_wire + p * ts_wire_record_size(has_rgb):
 *   i32 d_ij[2p], i32 d_ij[2p+1], f32 (float)d_cz[p], u8 d_stage[p],
 *   u8 flags (bit 0 = has_rgb), f32[64*64] heights_rel,
 *   u8[64*64*3] clip(round_half_even(f32(rgb*255)), 0, 255) if has_rgb.
 * d_out: B x 64 x 64 x 4 float32 (heights_rel, r, g, b) as ts_refine and
 * the bake leave it (16-byte aligned); d_wire 2-byte aligned.            */
size_t ts_wire_record_size(int has_rgb);
int ts_wire_heightmaps(const float* d_out, const double* d_cz, const int32_t* d_ij,
                       const uint8_t* d_stage, int has_rgb, int batch,
                       uint8_t* d_wire, void* stream);

/* ---- rendering (render.py:25-268, geometry.py:71-102) ------------------
 * A framebuffer is width x height uint64 min keys (EMPTY = all ones):
 * key = depth_key(eye depth) << 32 | 0xRRGGBBAA, merged with atomicMin, so
 * the image is independent of submission order.  The camera is the
 * reference's CameraState reduced on the host: position, the basis() unit
 * vectors, f = 1/tan(fov_y/2), f / aspect, near, far, viewport.          */
typedef struct ts_camera {
  double pos[3], right[3], up[3], fwd[3];
  double f, f_over_aspect, near, far;
  int32_t width, height;
} ts_camera;
/* rasterize_points (render.py:55-98): one fragment per in-frustum point;
 * d_rgb (n,3) float32 in [0,1] or NULL (every point grey_color, the
 * reference's pack_color(0.85 grey)).                                    */
int ts_render_points(const double* d_xyz, const float* d_rgb, int64_t n,
                     const ts_camera* cam, uint32_t grey_color, uint64_t* d_fb,
                     void* stream);
/* rasterize_heightmaps (render.py:101-239): patch_mesh triangles of each
 * refined patch (heights_rel P x 64 x 64 float32 + c_z, centres P x 2),
 * quad colours from rgb (P x 64 x 64 x 3, used where d_has_rgb[p]) or the
 * height shade; small / large triangle paths with identical per-pixel
 * arithmetic.  d_scratch: ts_render_heightmaps_scratch(P) bytes.         */
size_t ts_render_heightmaps_scratch(int n_patches);
int ts_render_heightmaps(const float* d_heights, const float* d_rgb,
                         const uint8_t* d_has_rgb, const double* d_center,
                         const double* d_cz, int n_patches, const ts_camera* cam,
                         uint64_t* d_fb, void* d_scratch, void* stream);
/* resolve (render.py:254-268): colour bytes of each key through the sRGB
 * table (the reference's _srgb_lut), background where empty; RGBA8.      */
typedef struct ts_srgb_lut {
  uint8_t v[256];
} ts_srgb_lut;
int ts_render_resolve(const uint64_t* d_fb, int64_t n_cells, const ts_srgb_lut* lut,
                      const uint8_t background[3], uint8_t* d_rgba, void* stream);

/* projected_bbox_area (geometry.py:128-164) of n boxes (n x 6 float64:
 * min xyz, max xyz) -> screen-space AABB area and diagonal, 0 for boxes
 * outside the frustum (the six inward planes of frustum_planes,
 * geometry.py:105-125, computed on the host).  The scheduler's viewpoint
 * priorities (engine.py:185-202) for every patch and tile in one launch. */
typedef struct ts_frustum {
  double plane[6][4];
} ts_frustum;
int ts_bbox_areas(const double* d_boxes, int64_t n, const ts_camera* cam,
                  const ts_frustum* frustum, double* d_area, double* d_diag,
                  void* stream);

/* ---- test hooks (host-callable, no GPU needed) ------------------------ */
/* Sign of the exact incircle / orientation determinants used by
 * ts_triangulate: returns -1, 0, +1.                                     */
int ts_incircle_sign(const double a[2], const double b[2], const double c[2],
                     const double d[2]);
int ts_orient_sign(const double a[2], const double b[2], const double c[2]);
/* The same predicates evaluated by device code: n cases of 8 doubles
 * (mode 0: orient of the first 6, mode 1: incircle of all 8).           */
int ts_predicates_device(const double* d_in, int64_t n, int mode,
                         int32_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TS_B200_H */
