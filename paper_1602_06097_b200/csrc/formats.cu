// formats.cu -- SURVEY 8(f) f3: the paper's binary matrix formats (Table
// `tab:bin_formats` P:241-270) decoded on the device into the CSR that gbla_splice / gbla_reduce
// take.  Readings (R20 + R23-R26): little-endian; Format 2 type code b & 7 = u | (v << 1)
// with data of 8 * 2^v bits (010 and the paper's own "011" both read as 16-bit), format version in
// b >> 24 (0 or 1 accepted); a column run of s > 1 columns from f is the colid slot pair (f, s), a
// single column f the one slot f | 2^31; polynomial j of length prow[j] starts at the sum of the
// earlier prow, row i carries polynomial polmap[i].
//
// Format 2 decoding is one pass over each section, HBM-bound:
//   row_ptr = exclusive scan of rows (u32 -> u64), pstart = exclusive scan of prow;
//   colid: slot j is a run length iff an odd number of unmasked slots precede it (pairs (f, s)
//   are the only unmasked slots; a masked slot after an odd count is an error) -- a prefix sum
//   of the unmasked flags; each slot then emits 1 (single), 0 (run head) or s (run length)
//   columns at the exclusive prefix sum of those counts;
//   values: one warp per row copies polynomial polmap[i] (widened / narrowed to u16).
// Input errors (counts that do not add up, a run without its length, a polynomial whose length is
// not the row's, a value outside [1, p)) are latched on the device and returned as GBLA_E_INVAL.
#include <string.h>

#include <cub/cub.cuh>

#include "internal.cuh"

namespace {

constexpr uint64_t MASK = 1ull << 31;
enum { FE_COUNT = 1, FE_RUN = 2, FE_POLY = 4, FE_VALUE = 8 };

__global__ void k_widen(int64_t n, const uint32_t *__restrict__ a, uint64_t *__restrict__ b)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
    else if (i == n) b[i] = 0;
}

// flag[j] = colid[j] is unmasked
__global__ void k_unmasked(int64_t k, const uint64_t *__restrict__ tok, uint64_t *__restrict__ flag)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) flag[j] = (tok[j] & MASK) ? 0 : 1;
    else if (j == k) flag[j] = 0;
}

// columns emitted by slot j (given the number of unmasked slots before it)
__global__ void k_slot_cols(int64_t k, const uint64_t *__restrict__ tok, const uint64_t *__restrict__ before,
                            uint64_t *__restrict__ cnt, uint32_t *__restrict__ err)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j > k) return;
    if (j == k) {                                  // the stream must end after a complete pair
        cnt[j] = 0;
        if (before[k] & 1) atomicOr(err, FE_RUN);
        return;
    }
    const uint64_t t = tok[j];
    const bool odd = before[j] & 1;
    if (t & MASK) {
        cnt[j] = 1;
        if (odd) atomicOr(err, FE_RUN);            // a single column where a run length belongs
    } else {
        cnt[j] = odd ? t : 0;                      // run length s, or run head f
        if (odd && t < 2) atomicOr(err, FE_RUN);   // runs are s > 1
    }
}

__global__ void k_emit_cols(int64_t k, uint64_t nnz, const uint64_t *__restrict__ tok,
                            const uint64_t *__restrict__ before, const uint64_t *__restrict__ pos,
                            uint32_t *__restrict__ col, uint32_t *__restrict__ err)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    const uint64_t t = tok[j];
    const uint64_t o = pos[j];
    if (t & MASK) {
        if (o < nnz) col[o] = (uint32_t)(t & ~MASK);
        else atomicOr(err, FE_COUNT);
    } else if (before[j] & 1) {
        const uint64_t f = tok[j - 1];
        if (o + t > nnz) { atomicOr(err, FE_COUNT); return; }
        for (uint64_t u = 0; u < t; u++) col[o + u] = (uint32_t)(f + u);
    }
}

// values of row i = polynomial polmap[i]; width = bytes per pdata element
__global__ void k_poly_vals(int64_t m, const uint64_t *__restrict__ rp, const uint32_t *__restrict__ polmap,
                            int64_t pnb, const uint32_t *__restrict__ prow, const uint64_t *__restrict__ pstart,
                            const uint8_t *__restrict__ pdata, int width, uint32_t p, uint16_t *__restrict__ val,
                            uint32_t *__restrict__ err)
{
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= m) return;
    const uint32_t j = polmap[i];
    const uint64_t s = rp[i], len = rp[i + 1] - s;
    if (j >= pnb || prow[j] != len) {
        if (lane == 0) atomicOr(err, FE_POLY);
        return;
    }
    const uint64_t q0 = pstart[j];
    uint32_t bad = 0;
    for (uint64_t r = lane; r < len; r += 32) {
        const uint8_t *e = pdata + (q0 + r) * width;
        uint64_t v = 0;
        for (int b = 0; b < width; b++) v |= (uint64_t)e[b] << (8 * b);
        if (v == 0 || v >= p) bad = 1;
        val[s + r] = (uint16_t)v;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, FE_VALUE);
}

template <class T>
gbla_status scan_excl(gbla_ctx ctx, cudaStream_t st, const T *in, T *out, int64_t n)
{
    size_t tb = 0;
    GBLA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)n, st));
    void *t = ctx_alloc(ctx, tb + 16, st);
    if (!t) { set_error("format decoding: scan workspace"); return GBLA_E_NOMEM; }
    const cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tb, in, out, (int)n, st);
    ctx_free(ctx, t, st);
    GBLA_CUDA_TRY(e);
    return GBLA_OK;
}

struct Sections {           // byte offsets of the Format 2 sections
    size_t rows, polmap, colid, prow, pdata, end;
};

static gbla_status parse_header(const uint8_t *b, size_t len, int format, gbla_file_info *fi, Sections *sec)
{
    memset(fi, 0, sizeof *fi);
    fi->format = format;
    auto rd32 = [&](size_t o) { uint32_t v; memcpy(&v, b + o, 4); return v; };
    auto rd64 = [&](size_t o) { uint64_t v; memcpy(&v, b + o, 8); return v; };
    if (format == 1) {
        if (len < 20) { set_error("format 1: truncated header (%zu bytes)", len); return GBLA_E_INVAL; }
        fi->m = rd32(0);
        fi->n = rd32(4);
        fi->p = rd32(8);
        fi->nnz = (int64_t)rd64(12);
        const size_t need = 20 + (size_t)fi->nnz * 6 + (size_t)fi->m * 4;
        if (fi->nnz < 0 || len != need) { set_error("format 1: %zu bytes, the header implies %zu", len, need); return GBLA_E_INVAL; }
        fi->typecode = 0b010;
        return GBLA_OK;
    }
    if (format != 2) { set_error("unknown format %d (1 or 2)", format); return GBLA_E_INVAL; }
    if (len < 28) { set_error("format 2: truncated header (%zu bytes)", len); return GBLA_E_INVAL; }
    const uint32_t bb = rd32(0);
    fi->typecode = bb & 7;
    fi->version = bb >> 24;
    if (fi->version > 1) { set_error("format 2: unknown version %u", fi->version); return GBLA_E_INVAL; }
    fi->m = rd32(4);
    fi->n = rd32(8);
    const uint64_t p64 = rd64(12);
    fi->nnz = (int64_t)rd64(20);
    if (p64 >= 65536) { set_error("format 2: p = %llu (this library: p < 2^16)", (unsigned long long)p64); return GBLA_E_DOMAIN; }
    fi->p = (uint32_t)p64;
    if (fi->m >= (1ll << 31)) { set_error("format 2: m >= 2^31"); return GBLA_E_INVAL; }
    size_t o = 28;
    sec->rows = o; o += (size_t)fi->m * 4;
    sec->polmap = o; o += (size_t)fi->m * 4;
    if (o + 8 > len) { set_error("format 2: truncated before k"); return GBLA_E_INVAL; }
    fi->k = (int64_t)rd64(o); o += 8;
    sec->colid = o; o += (size_t)fi->k * 8;
    if (o + 12 > len) { set_error("format 2: truncated before pnb"); return GBLA_E_INVAL; }
    fi->pnb = rd32(o); o += 4;
    fi->pnnz = (int64_t)rd64(o); o += 8;
    sec->prow = o; o += (size_t)fi->pnb * 4;
    sec->pdata = o;
    const int width = 1 << ((fi->typecode >> 1) & 3);
    o += (size_t)fi->pnnz * width;
    sec->end = o;
    if (o != len) { set_error("format 2: %zu bytes, the header implies %zu", len, o); return GBLA_E_INVAL; }
    return GBLA_OK;
}

}  // namespace

extern "C" gbla_status gbla_file_info_parse(const void *bytes, size_t len, int format, gbla_file_info *out)
{
    if (!bytes || !out) { set_error("gbla_file_info_parse: NULL argument"); return GBLA_E_INVAL; }
    Sections sec;
    return parse_header((const uint8_t *)bytes, len, format, out, &sec);
}

extern "C" gbla_status gbla_file_decode(gbla_ctx ctx, const void *bytes, size_t len, int format, uint64_t *row_ptr,
                                        uint32_t *col, uint16_t *val, void *stream)
{
    if (!ctx || !bytes || !row_ptr) { set_error("gbla_file_decode: NULL argument"); return GBLA_E_INVAL; }
    gbla_file_info fi;
    Sections sec;
    GBLA_TRY(parse_header((const uint8_t *)bytes, len, format, &fi, &sec));
    if (fi.nnz > 0 && (!col || !val)) { set_error("gbla_file_decode: NULL col / val"); return GBLA_E_INVAL; }
    GBLA_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const uint8_t *b = (const uint8_t *)bytes;
    const int64_t m = fi.m, nnz = fi.nnz;
    std::vector<void *> tmp;
    auto talloc = [&](size_t bytes_) -> void * {
        void *q = ctx_alloc(ctx, bytes_ + 16, st);
        if (q) tmp.push_back(q);
        return q;
    };
    gbla_status s = GBLA_OK;
    uint32_t *err = (uint32_t *)talloc(4);
    uint32_t *rows = (uint32_t *)talloc((size_t)m * 4);
    if (!err || !rows) s = GBLA_E_NOMEM;
    if (s == GBLA_OK) {
        cudaMemsetAsync(err, 0, 4, st);
        const size_t roff = format == 1 ? 20 + (size_t)nnz * 6 : sec.rows;
        if (m) cudaMemcpyAsync(rows, b + roff, (size_t)m * 4, cudaMemcpyHostToDevice, st);
        uint64_t *w = (uint64_t *)talloc((size_t)(m + 1) * 8);
        if (!w) s = GBLA_E_NOMEM;
        if (s == GBLA_OK) {
            k_widen<<<grid_for(m + 1, 256), 256, 0, st>>>(m, rows, w);
            note_launch();
            s = scan_excl<uint64_t>(ctx, st, w, row_ptr, m + 1);
        }
    }
    if (s == GBLA_OK && format == 1) {                     // data and cols are CSR already
        if (nnz) {
            cudaMemcpyAsync(val, b + 20, (size_t)nnz * 2, cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(col, b + 20 + (size_t)nnz * 2, (size_t)nnz * 4, cudaMemcpyHostToDevice, st);
        }
    } else if (s == GBLA_OK) {
        const int64_t k = fi.k, pnb = fi.pnb, pnnz = fi.pnnz;
        const int width = 1 << ((fi.typecode >> 1) & 3);
        uint32_t *polmap = (uint32_t *)talloc((size_t)m * 4);
        uint64_t *tok = (uint64_t *)talloc((size_t)k * 8);
        uint64_t *flag = (uint64_t *)talloc((size_t)(k + 1) * 8), *before = (uint64_t *)talloc((size_t)(k + 1) * 8);
        uint64_t *cnt = (uint64_t *)talloc((size_t)(k + 1) * 8), *pos = (uint64_t *)talloc((size_t)(k + 1) * 8);
        uint32_t *prow = (uint32_t *)talloc((size_t)pnb * 4);
        uint64_t *pw = (uint64_t *)talloc((size_t)(pnb + 1) * 8), *pstart = (uint64_t *)talloc((size_t)(pnb + 1) * 8);
        uint8_t *pdata = (uint8_t *)talloc((size_t)pnnz * width);
        if (!polmap || !tok || !flag || !before || !cnt || !pos || !prow || !pw || !pstart || !pdata) {
            set_error("gbla_file_decode: staging allocation failed");
            s = GBLA_E_NOMEM;
        }
        if (s == GBLA_OK) {
            if (m) cudaMemcpyAsync(polmap, b + sec.polmap, (size_t)m * 4, cudaMemcpyHostToDevice, st);
            if (k) cudaMemcpyAsync(tok, b + sec.colid, (size_t)k * 8, cudaMemcpyHostToDevice, st);
            if (pnb) cudaMemcpyAsync(prow, b + sec.prow, (size_t)pnb * 4, cudaMemcpyHostToDevice, st);
            if (pnnz) cudaMemcpyAsync(pdata, b + sec.pdata, (size_t)pnnz * width, cudaMemcpyHostToDevice, st);
            k_unmasked<<<grid_for(k + 1, 256), 256, 0, st>>>(k, tok, flag);
            k_widen<<<grid_for(pnb + 1, 256), 256, 0, st>>>(pnb, prow, pw);
            note_launch(2);
            s = scan_excl<uint64_t>(ctx, st, flag, before, k + 1);
        }
        if (s == GBLA_OK) {
            k_slot_cols<<<grid_for(k + 1, 256), 256, 0, st>>>(k, tok, before, cnt, err);
            note_launch();
            s = scan_excl<uint64_t>(ctx, st, cnt, pos, k + 1);
        }
        if (s == GBLA_OK) s = scan_excl<uint64_t>(ctx, st, pw, pstart, pnb + 1);
        uint64_t tot = 0;
        if (s == GBLA_OK) {
            k_emit_cols<<<grid_for(k, 256), 256, 0, st>>>(k, (uint64_t)nnz, tok, before, pos, col, err);
            if (m) k_poly_vals<<<grid_for(m * 32, 256), 256, 0, st>>>(m, row_ptr, polmap, pnb, prow, pstart, pdata, width,
                                                                      fi.p, val, err);
            note_launch(2);
            cudaMemcpyAsync(&tot, pos + k, 8, cudaMemcpyDeviceToHost, st);
        }
        if (s == GBLA_OK && cudaStreamSynchronize(st) == cudaSuccess && tot != (uint64_t)nnz) {
            set_error("format 2: colid decodes to %llu columns, nnz = %lld", (unsigned long long)tot, (long long)nnz);
            s = GBLA_E_INVAL;
        }
    }
    uint64_t rtot = 0;
    uint32_t e = 0;
    if (s == GBLA_OK) {
        cudaMemcpyAsync(&rtot, row_ptr + m, 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) {
            set_error("gbla_file_decode: %s", cudaGetErrorString(cudaGetLastError()));
            s = GBLA_E_CUDA;
        } else if (rtot != (uint64_t)nnz) {
            set_error("format %d: sum of row lengths %llu != nnz %lld", format, (unsigned long long)rtot, (long long)nnz);
            s = GBLA_E_INVAL;
        } else if (e) {
            set_error("format %d: malformed content (code 0x%x: 1 counts, 2 column runs, 4 polynomial lengths, 8 values)",
                      format, e);
            s = GBLA_E_INVAL;
        }
    }
    cudaStreamSynchronize(st);
    for (void *q : tmp) ctx_free(ctx, q, st);
    return s;
}
