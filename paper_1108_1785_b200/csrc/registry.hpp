// registry.hpp — host side of the site registry (replaces flowmon::SiteCatalog).
//
// Semantics follow site_catalog.hpp:29-97 / site_catalog.cpp (paths relative
// to /root/reference/proj/core): CIDRs expand into /24 tiles, prefixes longer
// than /24 round up to the enclosing /24, overlap with an existing site or
// within one registration is an error that leaves the registry unchanged,
// SiteId is the dense registration index.
//
// The representation is B200-first rather than a copy of the reference's
// open-addressing hash: the device needs a table that a whole CTA can keep
// in shared memory and probe with at most three dependent LDS, so the host
// compiles the /24 map into a two-level radix table (see compile_device_table).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace gnm {

struct Cidr {
    uint32_t addr = 0;
    int32_t prefix_len = 0;

    uint32_t network() const {
        const uint32_t mask = prefix_len == 0 ? 0 : ~uint32_t{0} << (32 - prefix_len);
        return addr & mask;
    }
    uint32_t first_prefix24() const { return network() & 0xFFFFFF00u; }
    uint32_t last_prefix24() const {
        if (prefix_len >= 24) return first_prefix24();
        const uint32_t span = 1u << (24 - prefix_len);
        return first_prefix24() + (span - 1) * 256u;
    }
};

// parse_ipv4 / Cidr::parse (site_catalog.cpp:10-66). Return false on
// malformed text; `err` receives the reference's message.
bool parse_ipv4(const std::string& text, uint32_t* out, std::string* err);
bool parse_cidr(const std::string& text, Cidr* out, std::string* err);
std::string format_ipv4(uint32_t ip);

// Device lookup table, one flat u32 array:
//   words [0, 4096)          : 2048 x {bitmap, rank} pairs over the 65536 /16
//                              blocks (bit set = the /16 holds a registered /24)
//   words [4096, 4096+N16)   : one node per non-empty /16, in address order:
//                              bit31 set -> every /24 of the block is site
//                              (node & 0x7FFFFFFF); else the word offset of a
//                              256-word leaf
//   leaves                   : 256 words per mixed /16, site per /24 or
//                              0xFFFFFFFF.
// lookup(ip): d = ip>>16; {bits,rank} = words[2*(d>>5)..]; miss unless bit
// d&31 is set; node = words[4096 + rank + popc(bits & below)];
// value = uniform ? node&0x7FFFFFFF : words[node + ((ip>>8)&255)].
//
// Site values are PACKED when the registry has fewer than 2^20 sites:
// bits 0..19 hold the SiteId and bits 20..30 a per-call hot slot (0 = cold),
// rewritten on the device before each accumulation (kernels.cu,
// k_table_slots). Larger registries store the plain 31-bit SiteId and run
// without hot slots (`packed` false).
struct DeviceTable {
    std::vector<uint32_t> words;
    uint32_t n_blocks16 = 0;
    uint32_t n_leaves = 0;
    uint32_t node_begin = 4096;  // first node word
    uint32_t leaf_begin = 4096;  // first leaf word
    bool packed = true;
};

constexpr uint32_t kNoSite = 0xFFFFFFFFu;
constexpr uint32_t kDirWords = 4096;
constexpr uint32_t kMaxSites = 0x3FFFFFFFu; // gnm_classify's 30-bit site field
constexpr uint32_t kPackedSiteBits = 20;
constexpr uint32_t kPackedSiteMask = (1u << kPackedSiteBits) - 1;

class Registry {
public:
    struct Site {
        uint32_t id;
        std::string name;
        std::vector<Cidr> cidrs;
    };

    // SiteCatalog::register_site (site_catalog.cpp:90-121). Returns 0, or
    // 2 (overlap) / 3 (invalid) / 1 (capacity) with `err` set.
    int register_site(const std::string& name, const std::vector<Cidr>& cidrs, uint32_t* out_id,
                      std::string* err);

    uint32_t lookup(uint32_t ip) const {
        auto it = index_.find(ip >> 8);
        return it == index_.end() ? kNoSite : it->second;
    }
    uint32_t sequential_lookup(uint32_t ip) const {
        const uint32_t p = ip & 0xFFFFFF00u;
        for (const auto& e : entries_)
            if (e.first == p) return e.second;
        return kNoSite;
    }

    const std::vector<Site>& sites() const { return sites_; }
    const std::vector<std::pair<uint32_t, uint32_t>>& entries() const { return entries_; }
    // Unique across all registries of the process (a fresh registry at a
    // recycled address never looks like one the device already holds).
    uint64_t version() const { return version_; }

    DeviceTable compile_device_table() const;

private:
    std::vector<Site> sites_;
    std::vector<std::pair<uint32_t, uint32_t>> entries_; // prefix24 -> site, insertion order
    std::unordered_map<uint32_t, uint32_t> index_;       // prefix24 >> 8 -> site
    uint64_t version_ = next_version();
    static uint64_t next_version();
};

} // namespace gnm
