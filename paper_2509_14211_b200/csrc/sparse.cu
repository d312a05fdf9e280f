// sparse.cu -- device helpers for structured vectors (PAPER.md:185
// SparseVector / BitSetVector, PAPER.md:236-246 representation choice).
//
//   SPARSE : nvals strictly ascending int32 indices + nvals values
//   BITSET : (n + 31) / 32 uint32 words (bit i of word i / 32 = entry i present) + n values
//
// Conversions keep index order, so every result is deterministic: sparse -> bitset is a scatter
// (distinct indices, no conflicts on values; bits set with atomicOr), bitset -> sparse is a
// per-word popcount + exclusive scan + scatter, and the index-driven compaction is CUB's stable
// DeviceSelect::Flagged.
#include <cub/cub.cuh>

#include "nbg_internal.hpp"

namespace nbg {

namespace {

int grid_of(int64_t work, int num_sms) {
    int64_t g = (work + 255) / 256;
    if (g > (int64_t)num_sms * 8) g = (int64_t)num_sms * 8;
    return (int)(g < 1 ? 1 : g);
}

__global__ void k_check_sparse(int64_t n, int64_t nv, const int32_t *idx, int *bad) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = idx[k];
        if (i < 0 || (int64_t)i >= n) atomicOr(bad, 2);
        if (k > 0 && idx[k - 1] >= i) atomicOr(bad, 1);
    }
}

template <typename W>
__global__ void k_sparse_scatter(int64_t nv, const int32_t *idx, const W *vals, uint32_t *bits, W *dense) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = idx[k];
        atomicOr(bits + (i >> 5), 1u << (i & 31));
        dense[i] = vals[k];
    }
}

__global__ void k_word_popc(int64_t nw, const uint32_t *bits, int64_t *cnt) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x)
        cnt[w] = __popc(bits[w]);
}

template <typename W>
__global__ void k_bits_gather(int64_t n, const uint32_t *bits, const W *dense, const int64_t *off, int32_t *oidx, W *ovals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t wd = bits[i >> 5];
        const int b = (int)(i & 31);
        if ((wd >> b) & 1u) {
            const int64_t pos = off[i >> 5] + __popc(wd & ((1u << b) - 1u));
            oidx[pos] = (int32_t)i;
            ovals[pos] = dense[i];
        }
    }
}

__global__ void k_full_bits(int64_t nw, int64_t n, uint32_t *bits) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rem = n - 32 * w;
        bits[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
    }
}

template <typename F>
void by_width(int type, F &&f) {
    switch (type_size(type)) {
        case 1: f((uint8_t *)nullptr); break;
        case 4: f((uint32_t *)nullptr); break;
        default: f((uint64_t *)nullptr); break;
    }
}

}  // namespace

int gpu_check_sparse(Ctx &c, int64_t n, int64_t nv, const int32_t *idx) {
    if (nv == 0) return 0;
    BufP bad = alloc_buf(c, 4);
    NBG_CUDA(cudaMemsetAsync(bad->d, 0, 4, c.stream));
    k_check_sparse<<<grid_of(nv, c.num_sms), 256, 0, c.stream>>>(n, nv, idx, (int *)bad->d);
    NBG_CUDA(cudaGetLastError());
    c.stats.kernels_launched++;
    int h = 0;
    NBG_CUDA(cudaMemcpyAsync(&h, bad->d, 4, cudaMemcpyDeviceToHost, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    return (h & 2) ? 2 : (h & 1);
}

void gpu_sparse_to_bitset(Ctx &c, int64_t n, int64_t nv, const int32_t *idx, const void *vals, int type, uint32_t *bits,
                          void *dense) {
    const int64_t nw = (n + 31) / 32;
    NBG_CUDA(cudaMemsetAsync(bits, 0, (size_t)nw * 4, c.stream));
    NBG_CUDA(cudaMemsetAsync(dense, 0, (size_t)n * type_size(type), c.stream));
    if (nv == 0) return;
    by_width(type, [&](auto *tag) {
        using W = std::remove_pointer_t<decltype(tag)>;
        k_sparse_scatter<W><<<grid_of(nv, c.num_sms), 256, 0, c.stream>>>(nv, idx, (const W *)vals, bits, (W *)dense);
    });
    NBG_CUDA(cudaGetLastError());
    c.stats.kernels_launched++;
}

int64_t gpu_bitset_to_sparse(Ctx &c, int64_t n, const uint32_t *bits, const void *dense, int type, BufP *oidx, BufP *ovals) {
    const int64_t nw = (n + 31) / 32;
    BufP cnt = alloc_buf(c, (size_t)(nw + 1) * 8), off = alloc_buf(c, (size_t)(nw + 1) * 8);
    NBG_CUDA(cudaMemsetAsync(cnt->d, 0, (size_t)(nw + 1) * 8, c.stream));
    if (nw) k_word_popc<<<grid_of(nw, c.num_sms), 256, 0, c.stream>>>(nw, bits, (int64_t *)cnt->d);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (const int64_t *)cnt->d, (int64_t *)off->d, (int64_t)(nw + 1), c.stream);
    BufP tmp = alloc_buf(c, std::max<size_t>(tb, 16));
    NBG_CUDA(cub::DeviceScan::ExclusiveSum(tmp->d, tb, (const int64_t *)cnt->d, (int64_t *)off->d, (int64_t)(nw + 1), c.stream));
    int64_t nv = 0;
    NBG_CUDA(cudaMemcpyAsync(&nv, (const int64_t *)off->d + nw, 8, cudaMemcpyDeviceToHost, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    *oidx = alloc_buf(c, (size_t)std::max<int64_t>(nv, 1) * 4);
    *ovals = alloc_buf(c, (size_t)std::max<int64_t>(nv, 1) * type_size(type));
    if (nv > 0) {
        by_width(type, [&](auto *tag) {
            using W = std::remove_pointer_t<decltype(tag)>;
            k_bits_gather<W><<<grid_of(n, c.num_sms), 256, 0, c.stream>>>(n, bits, (const W *)dense, (const int64_t *)off->d,
                                                                           (int32_t *)(*oidx)->d, (W *)(*ovals)->d);
        });
    }
    NBG_CUDA(cudaGetLastError());
    c.stats.kernels_launched += nv > 0 ? 3 : 2;
    return nv;
}

int64_t gpu_select_flagged(Ctx &c, int64_t m, const int32_t *idx, const void *vals, const uint8_t *flags, int type, BufP *oidx,
                           BufP *ovals) {
    BufP nsel = alloc_buf(c, 8);
    *oidx = alloc_buf(c, (size_t)std::max<int64_t>(m, 1) * 4);
    *ovals = alloc_buf(c, (size_t)std::max<int64_t>(m, 1) * type_size(type));
    NBG_CUDA(cudaMemsetAsync(nsel->d, 0, 8, c.stream));
    if (m > 0) {
        size_t tb = 0, tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, idx, flags, (int32_t *)(*oidx)->d, (int64_t *)nsel->d, m, c.stream);
        by_width(type, [&](auto *tag) {
            using W = std::remove_pointer_t<decltype(tag)>;
            cub::DeviceSelect::Flagged(nullptr, tb2, (const W *)vals, flags, (W *)(*ovals)->d, (int64_t *)nsel->d, m, c.stream);
        });
        BufP tmp = alloc_buf(c, std::max<size_t>(std::max(tb, tb2), 16));
        NBG_CUDA(cub::DeviceSelect::Flagged(tmp->d, tb, idx, flags, (int32_t *)(*oidx)->d, (int64_t *)nsel->d, m, c.stream));
        by_width(type, [&](auto *tag) {
            using W = std::remove_pointer_t<decltype(tag)>;
            NBG_CUDA(cub::DeviceSelect::Flagged(tmp->d, tb2, (const W *)vals, flags, (W *)(*ovals)->d, (int64_t *)nsel->d, m,
                                                c.stream));
        });
        c.stats.kernels_launched += 2;
    }
    int64_t nv = 0;
    NBG_CUDA(cudaMemcpyAsync(&nv, nsel->d, 8, cudaMemcpyDeviceToHost, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    return nv;
}

int64_t gpu_union_indices(Ctx &c, const std::vector<std::pair<const int32_t *, int64_t>> &lists, BufP *out) {
    int64_t tot = 0;
    for (auto &l : lists) tot += l.second;
    BufP cat = alloc_buf(c, (size_t)std::max<int64_t>(tot, 1) * 4), srt = alloc_buf(c, (size_t)std::max<int64_t>(tot, 1) * 4);
    int64_t off = 0;
    for (auto &l : lists) {
        if (l.second) NBG_CUDA(cudaMemcpyAsync((int32_t *)cat->d + off, l.first, (size_t)l.second * 4, cudaMemcpyDeviceToDevice, c.stream));
        off += l.second;
    }
    *out = alloc_buf(c, (size_t)std::max<int64_t>(tot, 1) * 4);
    BufP nsel = alloc_buf(c, 8);
    NBG_CUDA(cudaMemsetAsync(nsel->d, 0, 8, c.stream));
    if (tot > 0) {
        size_t tb = 0, tb2 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, (const uint32_t *)cat->d, (uint32_t *)srt->d, tot, 0, 32, c.stream);
        cub::DeviceSelect::Unique(nullptr, tb2, (const int32_t *)srt->d, (int32_t *)(*out)->d, (int64_t *)nsel->d, tot, c.stream);
        BufP tmp = alloc_buf(c, std::max<size_t>(std::max(tb, tb2), 16));
        NBG_CUDA(cub::DeviceRadixSort::SortKeys(tmp->d, tb, (const uint32_t *)cat->d, (uint32_t *)srt->d, tot, 0, 32, c.stream));
        NBG_CUDA(cub::DeviceSelect::Unique(tmp->d, tb2, (const int32_t *)srt->d, (int32_t *)(*out)->d, (int64_t *)nsel->d, tot,
                                           c.stream));
        c.stats.kernels_launched += 2;
    }
    int64_t nu = 0;
    NBG_CUDA(cudaMemcpyAsync(&nu, nsel->d, 8, cudaMemcpyDeviceToHost, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    return nu;
}

void gpu_bitset_full(Ctx &c, int64_t n, uint32_t *bits) {
    const int64_t nw = (n + 31) / 32;
    if (nw == 0) return;
    k_full_bits<<<grid_of(nw, c.num_sms), 256, 0, c.stream>>>(nw, n, bits);
    NBG_CUDA(cudaGetLastError());
    c.stats.kernels_launched++;
}

}  // namespace nbg
