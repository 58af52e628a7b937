// radix_sort.cu — hand-written stable LSD radix sort of (u64 key, u32 value)
// pairs on sm_100a.  8-bit digits; per pass: tile histograms (digit-major),
// a device-wide exclusive scan of the histogram (scan.cu, reduce-then-scan),
// and a scatter in which each tile ranks its keys stably with eight 1-bit
// block splits in shared memory.
// Used for tensor-id ordering of candidates (planner.py:283-284) and the
// plan-entry order (planner.py:360-361); only the bits that vary are sorted.
#include "common.cuh"
#include "block_scan.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"

namespace tio {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 4;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void __launch_bounds__(RS_THREADS)
rs_hist(const uint64_t *keys, int64_t n, int shift, int64_t *hist, int64_t ntiles) {
    pdl_wait();
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int i = 0; i < RS_ITEMS; ++i) {
        int64_t k = base + (int64_t)i * RS_THREADS + threadIdx.x;
        if (k < n) atomicAdd(&h[(keys[k] >> shift) & 255], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_THREADS)
rs_scatter(const uint64_t *kin, const uint32_t *vin, uint64_t *kout, uint32_t *vout, int64_t n,
           int shift, const int64_t *offs, int64_t ntiles) {
    pdl_wait();
    __shared__ uint64_t sk[2][RS_TILE];
    __shared__ uint32_t sv[2][RS_TILE];
    __shared__ uint32_t dstart[256];
    __shared__ int64_t sm[40];
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    const int64_t valid = n - base < RS_TILE ? n - base : RS_TILE;
    for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
        int64_t k = base + i;
        sk[0][i] = i < valid ? kin[k] : ~0ull;
        sv[0][i] = i < valid ? vin[k] : 0u;
    }
    if (threadIdx.x < 256) dstart[threadIdx.x] = 0;
    __syncthreads();
    int cur = 0;
    // eight stable 1-bit splits: thread t owns positions [t*ITEMS, t*ITEMS+ITEMS)
    for (int bit = 0; bit < 8; ++bit) {
        int zeros = 0;
        uint32_t bits[RS_ITEMS];
#pragma unroll
        for (int j = 0; j < RS_ITEMS; ++j) {
            bits[j] = (uint32_t)((sk[cur][threadIdx.x * RS_ITEMS + j] >> (shift + bit)) & 1u);
            zeros += bits[j] == 0;
        }
        int64_t total;
        int64_t zb = block_exclusive_sum<int64_t>(zeros, sm, &total);
        int zl = 0;
#pragma unroll
        for (int j = 0; j < RS_ITEMS; ++j) {
            int p = threadIdx.x * RS_ITEMS + j;
            int dst;
            if (bits[j] == 0) dst = (int)(zb + zl++);
            else dst = (int)(total + (p - (zb + zl)));
            sk[cur ^ 1][dst] = sk[cur][p];
            sv[cur ^ 1][dst] = sv[cur][p];
        }
        __syncthreads();
        cur ^= 1;
    }
    // first position of each digit in the sorted tile
    for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
        uint32_t d = (sk[cur][i] >> shift) & 255;
        if (i == 0 || ((sk[cur][i - 1] >> shift) & 255) != d) dstart[d] = i;
    }
    __syncthreads();
    // padded keys (all ones) sort to the end of digit 255; they are never written
    for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
        uint64_t key = sk[cur][i];
        uint32_t d = (key >> shift) & 255;
        int64_t rank = i - dstart[d];
        // count valid keys of digit d only: padded ones come after all valid ones
        int64_t dst = offs[(int64_t)d * ntiles + blockIdx.x] + rank;
        if (i < valid) {
            kout[dst] = key;
            vout[dst] = sv[cur][i];
        }
    }
}

int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp,
                     int64_t *hist, int64_t n, int bits, cudaStream_t stream, bool *result_in_tmp) {
    *result_in_tmp = false;
    if (n <= 1 || bits <= 0) return TIO_OK;
    const int64_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    uint64_t *ka = keys, *kb = keys_tmp;
    uint32_t *va = vals, *vb = vals_tmp;
    for (int shift = 0; shift < bits; shift += 8) {
        TIO_CUDA(launch_pdl(rs_hist, dim3((unsigned)ntiles), dim3(RS_THREADS), 0, stream, ka, n, shift, hist, ntiles));
        ::tio::count_launch();
        TIO_TRY(exclusive_scan(hist, hist, 256 * ntiles, hist + 256 * ntiles, nullptr, stream));
        TIO_CUDA(launch_pdl(rs_scatter, dim3((unsigned)ntiles), dim3(RS_THREADS), 0, stream, ka, va, kb, vb, n, shift,
                            hist, ntiles));
        ::tio::count_launch();
        TIO_CUDA(cudaGetLastError());
        uint64_t *tk = ka; ka = kb; kb = tk;
        uint32_t *tv = va; va = vb; vb = tv;
        *result_in_tmp = !*result_in_tmp;
    }
    return TIO_OK;
}

// histogram + the scan's tile totals
int64_t radix_hist_elems(int64_t n) {
    const int64_t m = 256 * ((n + RS_TILE - 1) / RS_TILE);
    return m + scan_tmp_elems(m) + 1;
}

}  // namespace tio
