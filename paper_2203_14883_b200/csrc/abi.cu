// abi.cu -- handle management, error reporting and the device gate of libtgl.so.
#include <cstdlib>

#include "common.cuh"
#include "tsindex.cuh"

namespace tgl {

int read_and_clear_gather_err(cudaStream_t st, int* bits);  // gather.cu
int read_and_clear_state_err(cudaStream_t st, int* bits);   // state.cu

int check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TGL_ECUDA;
    static int cached[64] = {0};  // 0 unknown, 1 ok, 2 not supported
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev] == 1 ? TGL_OK : TGL_ENOTSUP;
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return TGL_ECUDA;
    if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return TGL_ECUDA;
    const bool ok = major == 10 && minor == 0;  // the fatbin holds sm_100a SASS only
    if (dev >= 0 && dev < 64) cached[dev] = ok ? 1 : 2;
    return ok ? TGL_OK : TGL_ENOTSUP;
}

}  // namespace tgl

using namespace tgl;

extern "C" int tgl_abi_version(void) { return TGL_ABI_VERSION; }

extern "C" const char* tgl_strerror(int code) {
    switch (code) {
        case TGL_OK: return "ok";
        case TGL_EINVAL: return "invalid argument or non-finite / negative time";
        case TGL_ERANGE: return "node or row id out of range";
        case TGL_EUNSORTED: return "edge stream is not chronological";
        case TGL_ECAPACITY: return "output buffer smaller than tgl_sample_capacity()";
        case TGL_EWORKSPACE: return "workspace smaller than required";
        case TGL_ECUDA: return "CUDA runtime error";
        case TGL_ENCCL: return "collective error";
        case TGL_ENOTSUP: return "device is not sm_100 (B200)";
        default: return "unknown error";
    }
}

extern "C" int tgl_tcsr_wrap(const int64_t* indptr, const int32_t* nbr, const float* ts, const int32_t* eid,
                             const void* aux, size_t aux_bytes, int32_t n_nodes, int64_t n_stored,
                             tgl_tcsr** out) {
    if (!out || !indptr || n_nodes < 0 || n_stored < 0) return TGL_EINVAL;
    *out = nullptr;
    if (n_stored > 0 && (!nbr || !ts || !eid)) return TGL_EINVAL;
    if ((uint64_t)n_stored >= (1ull << 32)) return TGL_EINVAL;
    const AuxLayout lay = aux_layout((uint64_t)n_stored, (uint64_t)n_nodes);
    if (aux && aux_bytes < lay.bytes) return TGL_EWORKSPACE;
    int rc = check_device();
    if (rc) return rc;
    tgl_tcsr* g = static_cast<tgl_tcsr*>(calloc(1, sizeof(tgl_tcsr)));
    if (!g) return TGL_EINVAL;
    if (cudaMalloc(&g->err_dev, sizeof(int)) != cudaSuccess || cudaMemset(g->err_dev, 0, sizeof(int)) != cudaSuccess) {
        free(g);
        return TGL_ECUDA;
    }
    g->indptr = indptr;
    g->nbr = nbr;
    g->ts = ts;
    g->eid = eid;
    g->n_nodes = n_nodes;
    g->n_stored = n_stored;
    const char* ab = static_cast<const char*>(aux);
    g->index = aux ? reinterpret_cast<const float*>(ab + lay.index_off) : nullptr;
    g->n_levels = aux ? lay.index.n_levels : 0;
    for (int l = 0; l <= kMaxIndexLevels && l < 12; ++l) g->level_off[l] = lay.index.off[l];
    g->recs = aux ? static_cast<const void*>(ab + lay.rec_off) : nullptr;
    g->nodes = aux ? static_cast<const void*>(ab + lay.node_off) : nullptr;
    if (aux) {
        // the codec header written by the aux build (a synchronous read: the aux build has completed)
        uint32_t hdr[6] = {0, 0, 0, 0, 0, 0};
        if (cudaMemcpy(hdr, aux, sizeof(hdr), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaFree(g->err_dev);
            free(g);
            return TGL_ECUDA;
        }
        const bool bad = hdr[0] != kDictMagic || hdr[1] > (uint32_t)kMaxCodes || hdr[2] > 2 || hdr[3] > 32 ||
                         (hdr[2] == 2 ? (hdr[1] != 0 || hdr[4] > 32 || hdr[3] + hdr[4] > 64) : hdr[4] > 8);
        if (bad) {
            cudaFree(g->err_dev);
            free(g);
            return TGL_EINVAL;  // not a buffer filled by tgl_tcsr_build / tgl_tcsr_aux_build
        }
        if (hdr[1] > 0) {
            g->dict = aux;
            g->codes = reinterpret_cast<const uint8_t*>(ab + lay.code_off);
            g->n_codes = (int)hdr[1];
            g->packed = (int)hdr[2];
            g->bits_nbr = (int)hdr[3];
            g->bits_code = (int)hdr[4];
        } else if (hdr[2] == 2) {  // integer-time packed records
            g->packed = 2;
            g->bits_nbr = (int)hdr[3];
            g->bits_code = (int)hdr[4];
            g->eid_base0 = (int32_t)hdr[5];
        }
    }
    cudaGetDevice(&g->device);
    *out = g;
    return TGL_OK;
}

extern "C" int tgl_tcsr_set_node_base(tgl_tcsr* g, int64_t node_lo) {
    if (!g || node_lo < 0 || node_lo + g->n_nodes >= (int64_t(1) << 31)) return TGL_EINVAL;
    g->node_lo = node_lo;
    return TGL_OK;
}

extern "C" int tgl_tcsr_destroy(tgl_tcsr* g) {
    if (!g) return TGL_EINVAL;
    if (g->err_dev) cudaFree(g->err_dev);
    free(g);
    return TGL_OK;
}

extern "C" int tgl_tcsr_info(const tgl_tcsr* g, int32_t* n_nodes, int64_t* n_stored) {
    if (!g) return TGL_EINVAL;
    if (n_nodes) *n_nodes = g->n_nodes;
    if (n_stored) *n_stored = g->n_stored;
    return TGL_OK;
}

extern "C" int tgl_tcsr_codec(const tgl_tcsr* g, int32_t* n_codes, int32_t* packed) {
    if (!g) return TGL_EINVAL;
    if (n_codes) *n_codes = g->n_codes;
    if (packed) *packed = g->packed;
    return TGL_OK;
}

extern "C" int tgl_check(tgl_tcsr* g, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int bits = 0;
    if (g) {
        if (cudaMemcpyAsync(&bits, g->err_dev, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess) return TGL_ECUDA;
        if (cudaMemsetAsync(g->err_dev, 0, sizeof(int), st) != cudaSuccess) return TGL_ECUDA;
    } else {
        int b2 = 0;
        int rc = read_and_clear_gather_err(st, &bits);
        if (rc) return rc;
        rc = read_and_clear_state_err(st, &b2);
        if (rc) return rc;
        if (cudaStreamSynchronize(st) != cudaSuccess) return TGL_ECUDA;
        bits |= b2;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return TGL_ECUDA;
    return err_bits_to_code(bits);
}
