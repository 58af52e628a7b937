// cufile_probe.cu — can the SSD tier use cuFile on this box, and at what
// rate?  (SURVEY §8d "Link measurement": cuFileWrite / cuFileRead of 1 GiB,
// GDS vs compat mode.)  For each path: open (O_DIRECT if the filesystem takes
// it), register, write a 1 GiB device buffer with cuFileWrite, read it back
// with cuFileRead into a second buffer, compare, then the same through the
// stream-ordered cuFileWriteAsync / cuFileReadAsync.  One JSON line.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/micro/cufile_probe.cu \
//      -o tools/micro/cufile_probe -lcufile -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void fill(uint32_t *p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)(i * 2654435761u) ^ seed;
}

__global__ void cmp(const uint32_t *a, const uint32_t *b, size_t n, unsigned long long *bad) {
    unsigned long long c = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        c += a[i] != b[i];
    if (c) atomicAdd(bad, c);
}

int main(int argc, char **argv) {
    const size_t SZ = (argc > 2) ? (size_t)atoll(argv[2]) << 20 : (size_t)1 << 30;
    const char *path = argc > 1 ? argv[1] : "/tmp/tio_cufile_probe.bin";
    std::string out = "{\"path\": \"" + std::string(path) + "\", \"bytes\": " + std::to_string(SZ);
    fprintf(stderr, "[cufile_probe] driver open...\n");
    CUfileError_t st = cuFileDriverOpen();
    fprintf(stderr, "[cufile_probe] driver open rc %d\n", (int)st.err);
    out += ", \"driver_open\": " + std::to_string((int)st.err);
    CUfileDrvProps_t props;
    memset(&props, 0, sizeof(props));
    if (cuFileDriverGetProperties(&props).err == CU_FILE_SUCCESS) {
        out += ", \"nvfs_version\": \"" + std::to_string(props.nvfs.major_version) + "." +
               std::to_string(props.nvfs.minor_version) + "\"";
        out += ", \"dstatusflags\": " + std::to_string(props.nvfs.dstatusflags);
        out += ", \"dcontrolflags\": " + std::to_string(props.nvfs.dcontrolflags);
        out += ", \"allow_compat_mode\": " +
               std::string((props.nvfs.dcontrolflags >> CU_FILE_ALLOW_COMPAT_MODE) & 1 ? "true" : "false");
        out += ", \"fflags\": " + std::to_string(props.fflags);
    }
    int fd = open(path, O_CREAT | O_RDWR | O_DIRECT, 0644);
    bool direct = fd >= 0;
    if (fd < 0) fd = open(path, O_CREAT | O_RDWR, 0644);
    out += ", \"o_direct\": " + std::string(direct ? "true" : "false");
    if (fd < 0) {
        printf("%s, \"error\": \"open failed\"}\n", out.c_str());
        return 1;
    }
    CUfileDescr_t d;
    memset(&d, 0, sizeof(d));
    d.handle.fd = fd;
    d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
    CUfileHandle_t fh;
    fprintf(stderr, "[cufile_probe] handle register (o_direct %d)...\n", (int)direct);
    st = cuFileHandleRegister(&fh, &d);
    fprintf(stderr, "[cufile_probe] handle register rc %d\n", (int)st.err);
    out += ", \"handle_register\": " + std::to_string((int)st.err);
    if (st.err != CU_FILE_SUCCESS) {
        printf("%s}\n", out.c_str());
        close(fd);
        unlink(path);
        return 0;
    }
    uint32_t *a = nullptr, *b = nullptr;
    unsigned long long *bad = nullptr;
    cudaMalloc(&a, SZ);
    cudaMalloc(&b, SZ);
    cudaMalloc(&bad, 8);
    const size_t n = SZ / 4;
    fill<<<1184, 256>>>(a, n, 0x1234u);
    cudaMemset(b, 0, SZ);
    cudaDeviceSynchronize();
    const CUfileError_t rb = cuFileBufRegister(a, SZ, 0);
    const CUfileError_t rb2 = cuFileBufRegister(b, SZ, 0);
    out += ", \"buf_register\": [" + std::to_string((int)rb.err) + ", " + std::to_string((int)rb2.err) + "]";
    // synchronous API, best of 3
    double bw = 1e30, br = 1e30;
    ssize_t wr = 0, rd = 0;
    for (int r = 0; r < 3; ++r) {
        fprintf(stderr, "[cufile_probe] sync write/read %d...\n", r);
        double t0 = now();
        wr = cuFileWrite(fh, a, SZ, 0, 0);
        fsync(fd);
        double t1 = now();
        rd = cuFileRead(fh, b, SZ, 0, 0);
        double t2 = now();
        if (t1 - t0 < bw) bw = t1 - t0;
        if (t2 - t1 < br) br = t2 - t1;
    }
    cudaMemset(bad, 0, 8);
    cmp<<<1184, 256>>>(a, b, n, bad);
    unsigned long long hbad = 0;
    cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost);
    out += ", \"sync\": {\"written\": " + std::to_string(wr) + ", \"read\": " + std::to_string(rd) +
           ", \"write_gbs\": " + std::to_string(SZ / bw / 1e9) + ", \"read_gbs\": " + std::to_string(SZ / br / 1e9) +
           ", \"mismatched_words\": " + std::to_string(hbad) + "}";
    // stream-ordered API
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    fprintf(stderr, "[cufile_probe] stream API...\n");
    const CUfileError_t rs = cuFileStreamRegister((CUstream)s, 15);
    size_t size = SZ;
    off_t foff = 0, boff = 0;
    ssize_t nw = -1, nr = -1;
    fill<<<1184, 256, 0, s>>>(a, n, 0x9876u);
    cudaMemsetAsync(b, 0, SZ, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    cudaEventRecord(e0, s);
    const CUfileError_t aw = cuFileWriteAsync(fh, a, &size, &foff, &boff, &nw, (CUstream)s);
    cudaEventRecord(e1, s);
    const CUfileError_t ar = cuFileReadAsync(fh, b, &size, &foff, &boff, &nr, (CUstream)s);
    cudaEventRecord(e2, s);
    const cudaError_t se = cudaStreamSynchronize(s);
    float mw = 0, mr = 0;
    cudaEventElapsedTime(&mw, e0, e1);
    cudaEventElapsedTime(&mr, e1, e2);
    cudaMemset(bad, 0, 8);
    cmp<<<1184, 256>>>(a, b, n, bad);
    cudaMemcpy(&hbad, bad, 8, cudaMemcpyDeviceToHost);
    out += ", \"async\": {\"stream_register\": " + std::to_string((int)rs.err) + ", \"write_rc\": " +
           std::to_string((int)aw.err) + ", \"read_rc\": " + std::to_string((int)ar.err) + ", \"stream\": \"" +
           cudaGetErrorString(se) + "\", \"written\": " + std::to_string(nw) + ", \"read\": " + std::to_string(nr) +
           ", \"write_gbs\": " + std::to_string(mw > 0 ? SZ / (mw * 1e6) : 0.0) +
           ", \"read_gbs\": " + std::to_string(mr > 0 ? SZ / (mr * 1e6) : 0.0) +
           ", \"mismatched_words\": " + std::to_string(hbad) + "}";
    cuFileStreamDeregister((CUstream)s);
    cuFileBufDeregister(a);
    cuFileBufDeregister(b);
    cuFileHandleDeregister(fh);
    close(fd);
    unlink(path);
    cuFileDriverClose();
    printf("%s}\n", out.c_str());
    return 0;
}
