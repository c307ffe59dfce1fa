// layout.h -- device-resident CSR layout shared by the kernels and the host.
//
// The reference keeps CsrMatrix<MultiComponent<K>> as int64 indptr/indices
// plus K component planes (sparse.hpp:47-78).  On the device the same matrix
// is re-laid out once at upload:
//
//  * SHORT rows (len <= long_threshold) go to a SELL-C-sigma store: rows are
//    sorted by length (descending, stable) inside windows of `sigma` rows and
//    cut into slices of C rows (C = 32 real, 16 complex: one warp per slice,
//    one thread -- two for complex -- per row).  Element k of slot t of slice
//    s lives at slice_ptr[s] + k*C + t, so every per-k load of a warp is one
//    contiguous 128/256-byte segment.  Column indices are int32; each value
//    component is its own plane (SoA), planes [0,K) = re, [K,2K) = im.
//  * LONG rows keep the reference's row-contiguous CSR order in a separate
//    store, processed cooperatively (deterministic: one CTA per row with the
//    reference's serial add chains; fast: warp-sized chunks + ordered combine).
//
// Vectors stay AoS [n][K] (the memory image of std::vector<MultiComponent<K>>)
// so host buffers copy without repacking and a QD gather is one 32-byte
// sector.
#pragma once
#include <cstdint>

namespace mpsg {

struct SellView {
  int nslices;
  int C;                     // rows per slice (32 real, 16 complex)
  const int64_t* slice_ptr;  // [nslices+1] element offsets (multiples of C)
  const int* slot_row;       // [nslices*C] original row, -1 for padding
  const int* slot_len;       // [nslices*C] row length (0 for padding)
  const int* col;            // [elems] int32 columns (0 in padding)
  const double* val;         // [nplanes][elems]
  int64_t stride;            // elems (plane stride)
};

struct LongView {
  int nrows;                 // number of long rows
  const int* row;            // [nrows] original row ids
  const int64_t* ptr;        // [nrows+1] offsets into col/val
  const int* col;            // [lnnz]
  const double* val;         // [nplanes][lnnz]
  int64_t stride;            // lnnz
  // fast-mode chunking: warp w sums elements [chunk_beg[w], chunk_end[w]) of
  // long row chunk_row[w] into partial slot chunk_slot[w]; the slots of a row
  // are [chunk_first[r], chunk_first[r+1]) in row-position order.  Chunks are
  // ordered column-block-major (see capi.cu) so concurrently running warps
  // gather from one block of x at a time.
  int chunk;
  int nchunks;
  const int* chunk_row;      // [nchunks] long-row index
  const int64_t* chunk_beg;  // [nchunks] offsets into col/val
  const int64_t* chunk_end;  // [nchunks]
  const int* chunk_slot;     // [nchunks] partial slot
  const int* chunk_first;    // [nrows+1] first slot of each long row
  double* partial;           // [nchunks][nsum*K]
  unsigned* counter;         // [nrows] arrival counters (self-resetting)
};

}  // namespace mpsg
