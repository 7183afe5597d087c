// NVTX ranges for profilers (nsys / ncu --nvtx): one per flush, planned pass
// launch and exchange, in the "naqs_b200" domain; the payload is the pass
// index or the exchanged global bit.  Header-only NVTX v3: without an
// attached tool every call is a null-pointer check.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cstdint>

namespace nqe {

inline nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("naqs_b200");
    return d;
}

struct NvtxRange {
    explicit NvtxRange(const char* name, int64_t payload = -1) {
        nvtxEventAttributes_t a{};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        if (payload >= 0) {
            a.payloadType = NVTX_PAYLOAD_TYPE_INT64;
            a.payload.llValue = payload;
        }
        nvtxDomainRangePushEx(nvtx_domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace nqe
