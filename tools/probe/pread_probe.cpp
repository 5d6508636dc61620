// pread_probe.cpp — page-cache read throughput into pinned vs pageable buffers, 1..16 threads
// (the host feeder's ceiling for SSTATBIN file sources).  Build: g++ -O2 -std=c++17 -pthread
// pread_probe.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -o pread_probe
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "/dev/shm/pread_probe.bin";
    const size_t bytes = argc > 2 ? strtoull(argv[2], nullptr, 10) : (4ull << 30);
    {
        std::vector<char> blk(64 << 20, 1);
        FILE* f = fopen(path, "wb");
        for (size_t w = 0; w < bytes; w += blk.size()) fwrite(blk.data(), 1, blk.size(), f);
        fclose(f);
    }
    int fd = open(path, O_RDONLY);
    void* pinned = nullptr;
    cudaMallocHost(&pinned, bytes);
    void* pageable = malloc(bytes);
    memset(pageable, 0, bytes);
    memset(pinned, 0, bytes);
    for (int which = 0; which < 3; ++which) {
        char* dst = (char*)(which == 0 ? pinned : pageable);
        for (int T : {1, 4, 8, 16}) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            const size_t per = bytes / T;
            if (which < 2) {
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        size_t off = t * per, left = per;
                        while (left) {
                            ssize_t got = pread(fd, dst + off, left > (1 << 30) ? (1 << 30) : left, off);
                            if (got <= 0) break;
                            off += got;
                            left -= got;
                        }
                    });
            } else {  // mmap + memcpy into pinned
                char* m = (char*)mmap(nullptr, bytes, PROT_READ, MAP_SHARED | MAP_POPULATE, fd, 0);
                for (int t = 0; t < T; ++t) th.emplace_back([&, t] { memcpy((char*)pinned + t * per, m + t * per, per); });
                for (auto& x : th) x.join();
                th.clear();
                munmap(m, bytes);
            }
            for (auto& x : th) x.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            printf("%-22s threads=%2d: %.1f GB/s\n", which == 0 ? "pread -> pinned" : which == 1 ? "pread -> pageable" : "mmap+memcpy -> pinned", T, bytes / s / 1e9);
        }
    }
    unlink(path);
    return 0;
}
