// Ingest probe (diagnostics, not product): can the copy engines DMA straight from the page cache?
//   nvcc -O2 -o tools/_build/mmap_probe tools/mmap_probe.cu && tools/_build/mmap_probe <dir> [threads]
// A: cudaHostRegister(ReadOnly) of mmap'ed shard files, B: H2D from the registered mappings,
// C: both pipelined (register on host threads, copy each file as soon as it is registered),
// D: the current path for reference: pread into a pinned ring + H2D.
#include <cuda_runtime.h>
#include <dirent.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

struct F {
    std::string path;
    size_t len;
    void* map;
    size_t off;
};

int main(int argc, char** argv) {
    const std::string dir = argv[1];
    const int T = argc > 2 ? std::atoi(argv[2]) : 16;
    std::vector<F> fs;
    DIR* d = opendir(dir.c_str());
    while (dirent* e = readdir(d)) {
        std::string n = e->d_name;
        if (n.size() > 4 && n.substr(n.size() - 4) == ".csv") fs.push_back(F{dir + "/" + n, 0, nullptr, 0});
    }
    closedir(d);
    std::sort(fs.begin(), fs.end(), [](const F& a, const F& b) { return a.path < b.path; });
    size_t total = 0;
    for (auto& f : fs) {
        struct stat st;
        stat(f.path.c_str(), &st);
        f.len = st.st_size;
        f.off = total;
        total += f.len;
    }
    std::printf("%zu files, %.2f GB, %d threads\n", fs.size(), total / 1e9, T);
    {
        int ro = 0;
        cudaDeviceGetAttribute(&ro, cudaDevAttrHostRegisterReadOnlySupported, 0);
        int hr = 0;
        cudaDeviceGetAttribute(&hr, cudaDevAttrHostRegisterSupported, 0);
        std::printf("HostRegisterSupported %d ReadOnlySupported %d\n", hr, ro);
        const size_t pg = 4096, L = (fs[0].len + pg - 1) / pg * pg;
        struct V {
            const char* name;
            int prot, flags;
            unsigned reg;
        } vs[] = {{"shared ro, ReadOnly", PROT_READ, MAP_SHARED, cudaHostRegisterReadOnly},
                  {"shared ro, Default", PROT_READ, MAP_SHARED, cudaHostRegisterDefault},
                  {"shared ro, ReadOnly|Portable", PROT_READ, MAP_SHARED, cudaHostRegisterReadOnly | cudaHostRegisterPortable},
                  {"private rw, Default", PROT_READ | PROT_WRITE, MAP_PRIVATE, cudaHostRegisterDefault},
                  {"shared rw(O_RDWR), Default", PROT_READ | PROT_WRITE, MAP_SHARED, cudaHostRegisterDefault}};
        for (const V& v : vs) {
            int fd = open(fs[0].path.c_str(), (v.prot & PROT_WRITE) && v.flags == MAP_SHARED ? O_RDWR : O_RDONLY);
            void* p = mmap(nullptr, L, v.prot, v.flags | MAP_POPULATE, fd, 0);
            close(fd);
            double t0 = now();
            cudaError_t e = cudaHostRegister(p, L, v.reg);
            double t1 = now();
            std::printf("  %-32s %s (%.2f ms for %.1f MB)\n", v.name, cudaGetErrorString(e), (t1 - t0) * 1e3, L / 1e6);
            cudaGetLastError();
            if (e == cudaSuccess) cudaHostUnregister(p);
            munmap(p, L);
        }
        std::fflush(stdout);
    }
    if (argc > 3 && argv[3][0] == 'x') return 0;
    const bool only_d = argc > 3 && argv[3][0] == 'd';
    uint8_t* dev;
    CK(cudaMalloc(&dev, total + 64));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    auto map_all = [&]() {
        for (auto& f : fs) {
            int fd = open(f.path.c_str(), O_RDONLY);
            f.map = mmap(nullptr, f.len, PROT_READ, MAP_SHARED | MAP_POPULATE, fd, 0);
            close(fd);
        }
    };
    auto unmap_all = [&]() {
        for (auto& f : fs) munmap(f.map, f.len);
    };
    for (int rep = 0; rep < (only_d ? 0 : 2); ++rep) {
        double t0 = now();
        map_all();
        double t1 = now();
        std::atomic<size_t> nxt{0};
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i)
            th.emplace_back([&] {
                for (size_t k = nxt++; k < fs.size(); k = nxt++)
                    CK(cudaHostRegister(fs[k].map, fs[k].len, cudaHostRegisterReadOnly));
            });
        for (auto& t : th) t.join();
        double t2 = now();
        for (auto& f : fs)
            for (size_t a = 0; a < f.len; a += 32u << 20)
                CK(cudaMemcpyAsync(dev + f.off + a, static_cast<uint8_t*>(f.map) + a,
                                   std::min<size_t>(32u << 20, f.len - a), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        double t3 = now();
        for (auto& f : fs) CK(cudaHostUnregister(f.map));
        double t4 = now();
        unmap_all();
        std::printf("A/B mmap %.1f ms | register %.1f ms (%.1f GB/s) | H2D %.1f ms (%.1f GB/s) | unregister %.1f ms\n",
                    (t1 - t0) * 1e3, (t2 - t1) * 1e3, total / (t2 - t1) / 1e9, (t3 - t2) * 1e3,
                    total / (t3 - t2) / 1e9, (t4 - t3) * 1e3);
    }
    // C: pipelined
    for (int rep = 0; rep < (only_d ? 0 : 3); ++rep) {
        double t0 = now();
        std::vector<std::atomic<int>> ready(fs.size());
        for (auto& r : ready) r = 0;
        std::atomic<size_t> nxt{0};
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i)
            th.emplace_back([&] {
                for (size_t k = nxt++; k < fs.size(); k = nxt++) {
                    int fd = open(fs[k].path.c_str(), O_RDONLY);
                    fs[k].map = mmap(nullptr, fs[k].len, PROT_READ, MAP_SHARED | MAP_POPULATE, fd, 0);
                    close(fd);
                    CK(cudaHostRegister(fs[k].map, fs[k].len, cudaHostRegisterReadOnly));
                    ready[k] = 1;
                }
            });
        for (size_t k = 0; k < fs.size(); ++k) {
            while (!ready[k].load()) std::this_thread::yield();
            CK(cudaMemcpyAsync(dev + fs[k].off, fs[k].map, fs[k].len, cudaMemcpyHostToDevice, s));
        }
        CK(cudaStreamSynchronize(s));
        double t1 = now();
        for (auto& t : th) t.join();
        for (auto& f : fs) CK(cudaHostUnregister(f.map));
        unmap_all();
        double t2 = now();
        std::printf("C pipelined map+register+H2D %.1f ms (%.1f GB/s), unregister+unmap %.1f ms\n", (t1 - t0) * 1e3,
                    total / (t1 - t0) / 1e9, (t2 - t1) * 1e3);
    }
    // D: pread into a pinned ring (16 x 32 MB) + H2D
    {
        const size_t CH = 32u << 20;
        const int slots = 16;
        uint8_t* ring;
        CK(cudaHostAlloc(&ring, CH * slots, cudaHostAllocDefault));
        std::vector<cudaEvent_t> ev(slots);
        for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        struct C {
            size_t f, a, n;
        };
        std::vector<C> cs;
        for (size_t i = 0; i < fs.size(); ++i)
            for (size_t a = 0; a < fs[i].len; a += CH) cs.push_back(C{i, a, std::min(CH, fs[i].len - a)});
        for (int rep = 0; rep < 3; ++rep) {
            double t0 = now();
            std::vector<std::atomic<int>> ready(cs.size());
            for (auto& r : ready) r = 0;
            std::atomic<size_t> nxt{0}, enq{0};
            std::vector<std::thread> th;
            for (int i = 0; i < T; ++i)
                th.emplace_back([&] {
                    for (size_t k = nxt++; k < cs.size(); k = nxt++) {
                        while (k >= static_cast<size_t>(slots) && enq.load() <= k - slots) std::this_thread::yield();
                        CK(cudaEventSynchronize(ev[k % slots]));
                        int fd = open(fs[cs[k].f].path.c_str(), O_RDONLY);
                        size_t got = 0;
                        while (got < cs[k].n) got += pread(fd, ring + (k % slots) * CH + got, cs[k].n - got, cs[k].a + got);
                        close(fd);
                        ready[k] = 1;
                    }
                });
            for (size_t k = 0; k < cs.size(); ++k) {
                while (!ready[k].load()) std::this_thread::yield();
                CK(cudaMemcpyAsync(dev + fs[cs[k].f].off + cs[k].a, ring + (k % slots) * CH, cs[k].n,
                                   cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(ev[k % slots], s));
                enq = k + 1;
            }
            CK(cudaStreamSynchronize(s));
            double t1 = now();
            for (auto& t : th) t.join();
            std::printf("D pread ring + H2D %.1f ms (%.1f GB/s)\n", (t1 - t0) * 1e3, total / (t1 - t0) / 1e9);
        }
    }
    return 0;
}
