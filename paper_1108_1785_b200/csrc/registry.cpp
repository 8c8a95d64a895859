// registry.cpp — host registry: CIDR parsing, /24 expansion, overlap checks
// and the device-table compiler. See registry.hpp.
#include "registry.hpp"

#include <algorithm>
#include <atomic>
#include <cctype>
#include <map>

namespace gnm {

uint64_t Registry::next_version() {
    static std::atomic<uint64_t> counter{0};
    return ++counter;
}


// parse_ipv4, site_catalog.cpp:10-40: exactly four dot-separated decimal
// octets, each 1-3 digits and <= 255, nothing trailing.
bool parse_ipv4(const std::string& text, uint32_t* out, std::string* err) {
    uint32_t ip = 0;
    size_t pos = 0;
    for (int octet = 0; octet < 4; ++octet) {
        if (pos >= text.size() || !std::isdigit(static_cast<unsigned char>(text[pos]))) {
            if (err) *err = "bad IPv4 address: " + text;
            return false;
        }
        uint32_t value = 0;
        size_t digits = 0;
        while (pos < text.size() && std::isdigit(static_cast<unsigned char>(text[pos]))) {
            value = value * 10 + static_cast<uint32_t>(text[pos] - '0');
            ++pos;
            if (++digits > 3 || value > 255) {
                if (err) *err = "bad IPv4 address: " + text;
                return false;
            }
        }
        ip = ip << 8 | value;
        if (octet < 3) {
            if (pos >= text.size() || text[pos] != '.') {
                if (err) *err = "bad IPv4 address: " + text;
                return false;
            }
            ++pos;
        }
    }
    if (pos != text.size()) {
        if (err) *err = "bad IPv4 address: " + text;
        return false;
    }
    *out = ip;
    return true;
}

// Cidr::parse, site_catalog.cpp:48-66: "<ipv4>/<len>", len one or two
// digits in 1..32.
bool parse_cidr(const std::string& text, Cidr* out, std::string* err) {
    const size_t slash = text.find('/');
    if (slash == std::string::npos || slash + 1 >= text.size()) {
        if (err) *err = "missing prefix length: " + text;
        return false;
    }
    Cidr c;
    if (!parse_ipv4(text.substr(0, slash), &c.addr, err)) return false;
    const std::string len = text.substr(slash + 1);
    if (len.size() > 2 || len.empty() || !std::isdigit(static_cast<unsigned char>(len[0])) ||
        (len.size() == 2 && !std::isdigit(static_cast<unsigned char>(len[1])))) {
        if (err) *err = "bad prefix length: " + text;
        return false;
    }
    c.prefix_len = std::stoi(len);
    if (c.prefix_len < 1 || c.prefix_len > 32) {
        if (err) *err = "prefix length out of range: " + text;
        return false;
    }
    *out = c;
    return true;
}

std::string format_ipv4(uint32_t ip) {
    return std::to_string(ip >> 24) + "." + std::to_string(ip >> 16 & 0xFF) + "." +
           std::to_string(ip >> 8 & 0xFF) + "." + std::to_string(ip & 0xFF);
}

// register_site, site_catalog.cpp:90-121. The reference checks each produced
// /24 with a linear sequential_lookup (O(entries)); the hash index gives the
// same answer in O(1).
int Registry::register_site(const std::string& name, const std::vector<Cidr>& cidrs,
                            uint32_t* out_id, std::string* err) {
    if (sites_.size() >= kMaxSites) {
        if (err) *err = "registry full";
        return 1;
    }
    const uint32_t id = static_cast<uint32_t>(sites_.size());
    std::vector<uint32_t> produced;
    for (const Cidr& c : cidrs) {
        if (c.prefix_len < 0 || c.prefix_len > 32) {
            if (err) *err = "prefix length out of range";
            return 3;
        }
        for (uint64_t p = c.first_prefix24(); p <= c.last_prefix24(); p += 256)
            produced.push_back(static_cast<uint32_t>(p));
    }
    for (uint32_t p : produced) {
        auto it = index_.find(p >> 8);
        if (it != index_.end()) {
            if (err)
                *err = format_ipv4(p) + "/24 already belongs to site '" + sites_[it->second].name + "'";
            return 2;
        }
    }
    std::vector<uint32_t> sorted = produced;
    std::sort(sorted.begin(), sorted.end());
    const auto dup = std::adjacent_find(sorted.begin(), sorted.end());
    if (dup != sorted.end()) {
        if (err) *err = format_ipv4(*dup) + "/24 produced twice by '" + name + "'";
        return 2;
    }
    sites_.push_back(Site{id, name, cidrs});
    for (uint32_t p : produced) {
        entries_.emplace_back(p, id);
        index_.emplace(p >> 8, id);
    }
    version_ = next_version();
    *out_id = id;
    return 0;
}

DeviceTable Registry::compile_device_table() const {
    // Group /24 entries by /16 block, in address order.
    std::map<uint32_t, std::vector<std::pair<uint32_t, uint32_t>>> blocks; // d16 -> (octet3, site)
    for (const auto& [p24, site] : entries_) blocks[p24 >> 16].emplace_back((p24 >> 8) & 0xFF, site);

    DeviceTable t;
    t.n_blocks16 = static_cast<uint32_t>(blocks.size());
    std::vector<uint32_t> nodes;
    std::vector<uint32_t> leaves;
    std::vector<uint32_t> bits(2048, 0);
    for (const auto& [d, list] : blocks) {
        bits[d >> 5] |= 1u << (d & 31);
        bool uniform = list.size() == 256;
        for (const auto& e : list) uniform = uniform && e.second == list.front().second;
        if (uniform) {
            nodes.push_back(0x80000000u | list.front().second);
        } else {
            const uint32_t leaf_off = static_cast<uint32_t>(leaves.size()); // fixed up below
            nodes.push_back(leaf_off);
            leaves.resize(leaves.size() + 256, kNoSite);
            for (const auto& e : list) leaves[leaf_off + e.first] = e.second;
            ++t.n_leaves;
        }
    }
    const uint32_t leaf_base = kDirWords + static_cast<uint32_t>(nodes.size());
    t.node_begin = kDirWords;
    t.leaf_begin = leaf_base;
    t.packed = sites_.size() <= kPackedSiteMask;
    for (uint32_t& n : nodes)
        if (!(n & 0x80000000u)) n += leaf_base;
    t.words.assign(kDirWords, 0);
    uint32_t rank = 0;
    for (uint32_t w = 0; w < 2048; ++w) {
        t.words[2 * w] = bits[w];
        t.words[2 * w + 1] = rank;
        rank += static_cast<uint32_t>(__builtin_popcount(bits[w]));
    }
    t.words.insert(t.words.end(), nodes.begin(), nodes.end());
    t.words.insert(t.words.end(), leaves.begin(), leaves.end());
    return t;
}

} // namespace gnm
