// Zero-copy file feed probe: can page-cache pages of a /dev/shm file be registered with CUDA fast
// enough (several threads, slot-sized windows) to DMA a file to the GPU at the PCIe link rate
// without the feeder's pread copy?
//   nvcc -O2 -o register_mt register_mt.cu -lpthread && ./register_mt <GB> [window MiB]
// 1. a file of <GB> GB in /dev/shm, mapped PROT_READ / MAP_SHARED
// 2. register/unregister every window with T = 1, 4, 8, 16 threads (cudaHostRegisterReadOnly)
// 3. pipelined: T threads register windows ahead of a copy stream that DMAs each registered window
//    to one device buffer; windows unregistered after their copy.  End-to-end GB/s.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));          \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IOLBF, 0);
    const double gb = argc > 1 ? atof(argv[1]) : 8.0;
    const bool rw = argc > 3 && argv[3][0] == 'w';  // map PROT_READ | PROT_WRITE (file opened O_RDWR)
    const size_t win = (argc > 2 ? atoi(argv[2]) : 256) << 20;
    const size_t bytes = (size_t)(gb * 1e9) / win * win;
    const char* path = "/dev/shm/register_mt.bin";
    {
        int fd = open(path, O_CREAT | O_TRUNC | O_RDWR, 0644);
        std::vector<char> buf(64 << 20);
        for (size_t i = 0; i < buf.size(); ++i) buf[i] = (char)(i * 131);
        for (size_t off = 0; off < bytes; off += buf.size())
            if (write(fd, buf.data(), std::min(buf.size(), bytes - off)) < 0) return 1;
        close(fd);
    }
    int fd = open(path, rw ? O_RDWR : O_RDONLY);
    char* map = (char*)mmap(nullptr, bytes, rw ? PROT_READ | PROT_WRITE : PROT_READ, MAP_SHARED, fd, 0);
    if (map == MAP_FAILED) return 2;
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    const size_t nwin = bytes / win;
    printf("file %.1f GB, %zu windows of %zu MiB, mapping %s\n", bytes / 1e9, nwin, win >> 20, rw ? "RW" : "read-only");
    {
        cudaError_t e = cudaHostRegister(map, win, cudaHostRegisterReadOnly);
        printf("first register: %s\n", cudaGetErrorString(e));
        if (e != cudaSuccess) return 4;
        cudaHostUnregister(map);
    }

    for (int T : {1, 4, 8, 16}) {
        std::atomic<size_t> next{0};
        std::atomic<int> bad{0};
        double t0 = now();
        std::vector<std::thread> th;
        for (int k = 0; k < T; ++k)
            th.emplace_back([&] {
                for (size_t w; (w = next++) < nwin;)
                    if (cudaHostRegister(map + w * win, win, cudaHostRegisterReadOnly) != cudaSuccess) bad++;
            });
        for (auto& t : th) t.join();
        double t1 = now();
        th.clear();
        next = 0;
        for (int k = 0; k < T; ++k)
            th.emplace_back([&] {
                for (size_t w; (w = next++) < nwin;)
                    if (cudaHostUnregister(map + w * win) != cudaSuccess) bad++;
            });
        for (auto& t : th) t.join();
        double t2 = now();
        printf("threads=%2d register %.1f GB/s  unregister %.1f GB/s  errors %d\n", T, bytes / (t1 - t0) / 1e9,
               bytes / (t2 - t1) / 1e9, bad.load());
        cudaGetLastError();
    }

    // pipelined feed: registrars fill a queue of registered windows, the copier DMAs them
    void* dev = nullptr;
    CK(cudaMalloc(&dev, win * 4));
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int T : {4, 8, 16}) {
        for (int ahead : {4, 8}) {
            std::vector<std::atomic<int>> ready(nwin);
            for (auto& r : ready) r = 0;
            std::atomic<size_t> next{0};
            std::atomic<size_t> released{0};  // windows whose copy finished (bounded look-ahead)
            double t0 = now();
            std::vector<std::thread> th;
            for (int k = 0; k < T; ++k)
                th.emplace_back([&] {
                    for (size_t w; (w = next++) < nwin;) {
                        while (w >= released.load() + ahead) std::this_thread::yield();
                        ready[w] = cudaHostRegister(map + w * win, win, cudaHostRegisterReadOnly) == cudaSuccess ? 1 : -1;
                    }
                });
            std::vector<cudaEvent_t> ev(nwin);
            for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            size_t done = 0;
            for (size_t w = 0; w < nwin; ++w) {
                while (ready[w].load() == 0) {  // release finished copies while the window is pinned
                    while (done < w && cudaEventQuery(ev[done]) == cudaSuccess) {
                        cudaHostUnregister(map + done * win);
                        released = ++done;
                    }
                    std::this_thread::yield();
                }
                if (ready[w] < 0) { printf("register failed\n"); exit(3); }
                CK(cudaMemcpyAsync((char*)dev + (w % 4) * win, map + w * win, win, cudaMemcpyHostToDevice, cs));
                CK(cudaEventRecord(ev[w], cs));
                while (done < w && cudaEventQuery(ev[done]) == cudaSuccess) {
                    cudaHostUnregister(map + done * win);
                    released = ++done;
                }
            }
            CK(cudaStreamSynchronize(cs));
            for (; done < nwin; ++done) cudaHostUnregister(map + done * win);
            released = done;
            double t1 = now();
            for (auto& t : th) t.join();
            for (auto& e : ev) cudaEventDestroy(e);
            printf("pipelined threads=%2d ahead=%d: %.1f GB/s end to end\n", T, ahead, bytes / (t1 - t0) / 1e9);
        }
    }
    munmap(map, bytes);
    close(fd);
    unlink(path);
    return 0;
}
