// csr.cuh -- shared device-graph helpers (definitions in csr.cu).
#pragma once
#include "common.cuh"

namespace plv {

template <class K, class V>
void sort_pairs(const K *kin, K *kout, const V *vin, V *vout, int64_t n, int begin_bit,
                int end_bit, cudaStream_t s);
int64_t select_flagged_index(const uint8_t *flags, int64_t n, int64_t *out, cudaStream_t s);
int64_t select_flagged_index32(const uint8_t *flags, int64_t n, int32_t *out, cudaStream_t s);
void offsets_from_degrees(const int32_t *deg, int64_t n, int64_t *off, cudaStream_t s);
void row_index(const int64_t *off, int64_t n, int64_t nnz, int32_t *rowidx, cudaStream_t s);
void iota_i32(int32_t *p, int64_t n, cudaStream_t s);
void gather_i32(const int32_t *src, const int32_t *idx, int64_t n, int32_t *out, cudaStream_t s);

void csr_from_merged(const int32_t *a, const int32_t *b, const double *w, int64_t M, int64_t n,
                     int64_t merged, int64_t *off, int32_t *nbr, double *wts, double *selfw,
                     double *k, int64_t *info_h, double *m_h, cudaStream_t s);
void csr_build(const int32_t *u, const int32_t *v, const double *w, int64_t R, int64_t n,
               int64_t *off, int32_t *nbr, double *wts, double *selfw, double *k,
               int64_t *info_h, double *m_h, cudaStream_t s);
int64_t edge_records(const int64_t *off, const int32_t *nbr, const double *wts, int64_t n,
                     int32_t *ra, int32_t *rb, double *rw, cudaStream_t s);

}  // namespace plv
