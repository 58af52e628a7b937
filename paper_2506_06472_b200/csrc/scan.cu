// scan.cu — device-wide exclusive scan of int64 (reduce-then-scan, 3 launches)
// and flag compaction, used by planner setup/finalize.
#include "common.cuh"
#include "block_scan.cuh"
#include "scan.cuh"

namespace tio {

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

// out[i] = exclusive prefix within the tile; tot[tile] = tile sum
__global__ void __launch_bounds__(SC_THREADS)
scan_tiles(const int64_t *in, int64_t *out, int64_t n, int64_t *tot) {
    pdl_wait();
    __shared__ int64_t sm[40];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_ITEMS;
    int64_t v[SC_ITEMS];
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j) {
        v[j] = base + j < n ? in[base + j] : 0;
        s += v[j];
    }
    int64_t total;
    int64_t run = block_exclusive_sum<int64_t>(s, sm, &total);
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j) {
        if (base + j < n) out[base + j] = run;
        run += v[j];
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024)
scan_totals(int64_t *tot, int64_t m, int64_t *grand) {
    pdl_wait();
    __shared__ int64_t sm[40];
    const int64_t per = (m + blockDim.x - 1) / blockDim.x;
    const int64_t b0 = threadIdx.x * per;
    const int64_t b1 = b0 + per < m ? b0 + per : m;
    int64_t s = 0;
    for (int64_t i = b0; i < b1; ++i) s += tot[i];
    int64_t total;
    int64_t run = block_exclusive_sum<int64_t>(s, sm, &total);
    for (int64_t i = b0; i < b1; ++i) {
        int64_t v = tot[i];
        tot[i] = run;
        run += v;
    }
    if (threadIdx.x == 0 && grand) *grand = total;
}

__global__ void __launch_bounds__(SC_THREADS)
scan_add(int64_t *out, int64_t n, const int64_t *tot) {
    pdl_wait();
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_ITEMS;
    const int64_t add = tot[blockIdx.x];
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j)
        if (base + j < n) out[base + j] += add;
}

int64_t scan_tmp_elems(int64_t n) { return (n + SC_TILE - 1) / SC_TILE + 1; }

int exclusive_scan(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, int64_t *grand,
                   cudaStream_t stream) {
    if (n <= 0) {
        if (grand) TIO_CUDA(cudaMemsetAsync(grand, 0, sizeof(int64_t), stream));
        return TIO_OK;
    }
    const int64_t tiles = (n + SC_TILE - 1) / SC_TILE;
    TIO_CUDA(launch_pdl(scan_tiles, dim3((unsigned)tiles), dim3(SC_THREADS), 0, stream, in, out, n, tmp));
    ::tio::count_launch();
    TIO_CUDA(launch_pdl(scan_totals, dim3(1), dim3(1024), 0, stream, tmp, tiles, grand));
    ::tio::count_launch();
    TIO_CUDA(launch_pdl(scan_add, dim3((unsigned)tiles), dim3(SC_THREADS), 0, stream, out, n, (const int64_t *)tmp));
    ::tio::count_launch();
    TIO_CUDA(cudaGetLastError());
    return TIO_OK;
}

}  // namespace tio
