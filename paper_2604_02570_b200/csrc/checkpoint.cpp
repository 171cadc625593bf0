// checkpoint.cpp -- reader of the reference's checkpoint directories
// (wsvd::ckpt, src/checkpoint.cpp:168-333) into device layers: the bridge
// from real WSVD artefacts (not random-init factors) to the kernels
// (SURVEY.md 8(f) row 2).
//
// Format (schema "wsvd-checkpoint-v1", checkpoint.cpp:168-247):
//   manifest.json   {schema, stage, model{embed_dim, head_dim, n_heads,
//                    n_layers, ...}, weights{name: file}, factors[{layer, role,
//                    head, rank, a, b}], weight_bits, activation_bits,
//                    input_rotation, quantized[{layer, role, head, rank,
//                    a{values, scales, clip, bits}, b{...}, s2_skew}]}
//   *.wsvd          WSVDMAT1: magic, u64 rows, u64 cols, fp64 row-major
//                    little-endian (matrix.cpp:251-284)
//   *.i8            WSVDI8T1: magic, u64 rows, u64 cols, int8 row-major
//                    (checkpoint.cpp:110-146)
// Quantised factors are stored already rotated, Q(S1 A S2^T) and Q(S2 B)
// (quant.cpp:344-358), with S1 = hadamard(E) ("input_rotation": "hadamard"),
// which is what wsvd_layer_set_head_quantized expects with act_rotation = 1.
//
// The JSON reader below accepts the subset the reference writes (objects,
// arrays, strings, numbers, literals); malformed files map to WSVD_EIO like
// the reference's IoError (checkpoint.cpp:45-49).
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/wsvd_b200.h"

namespace {

thread_local std::string g_ckpt_err;

struct IoErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ JSON --
struct JVal {
    enum Type { Null, Bool, Num, Str, Arr, Obj } t = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;

    const JVal* find(const char* key) const {
        if (t != Obj) return nullptr;
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
    const JVal& at(const char* key) const {
        const JVal* v = find(key);
        if (!v) throw IoErr(std::string("manifest: missing key '") + key + "'");
        return *v;
    }
    long long integer() const {
        if (t != Num || std::floor(num) != num) throw IoErr("manifest: expected an integer");
        return static_cast<long long>(num);
    }
    const std::string& string() const {
        if (t != Str) throw IoErr("manifest: expected a string");
        return str;
    }
};

class JParser {
  public:
    explicit JParser(const std::string& s) : s_(s) {}
    JVal parse() {
        JVal v = value();
        ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

  private:
    const std::string& s_;
    size_t i_ = 0;

    [[noreturn]] void fail(const char* what) const {
        throw IoErr(std::string("manifest: malformed JSON (") + what + " at byte " + std::to_string(i_) + ")");
    }
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
    }
    char peek() {
        ws();
        if (i_ >= s_.size()) fail("unexpected end");
        return s_[i_];
    }
    void expect(char c) {
        if (peek() != c) fail("unexpected character");
        ++i_;
    }
    JVal value() {
        const char c = peek();
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            JVal v;
            v.t = JVal::Str;
            v.str = string();
            return v;
        }
        if (s_.compare(i_, 4, "true") == 0) return i_ += 4, literal(JVal::Bool, true);
        if (s_.compare(i_, 5, "false") == 0) return i_ += 5, literal(JVal::Bool, false);
        if (s_.compare(i_, 4, "null") == 0) return i_ += 4, literal(JVal::Null, false);
        return number();
    }
    static JVal literal(JVal::Type t, bool b) {
        JVal v;
        v.t = t;
        v.b = b;
        return v;
    }
    JVal number() {
        const char* p = s_.c_str() + i_;
        char* end = nullptr;
        const double d = std::strtod(p, &end);
        if (end == p) fail("expected a value");
        i_ += static_cast<size_t>(end - p);
        JVal v;
        v.t = JVal::Num;
        v.num = d;
        return v;
    }
    std::string string() {
        expect('"');
        std::string out;
        while (true) {
            if (i_ >= s_.size()) fail("unterminated string");
            const char c = s_[i_++];
            if (c == '"') break;
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (i_ >= s_.size()) fail("bad escape");
            const char e = s_[i_++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    if (i_ + 4 > s_.size()) fail("bad \\u escape");
                    const unsigned cp = static_cast<unsigned>(std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16));
                    i_ += 4;
                    if (cp < 0x80) {
                        out.push_back(static_cast<char>(cp));
                    } else if (cp < 0x800) {
                        out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    } else {
                        out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    }
                    break;
                }
                default: fail("bad escape");
            }
        }
        return out;
    }
    JVal array() {
        expect('[');
        JVal v;
        v.t = JVal::Arr;
        if (peek() == ']') return ++i_, v;
        while (true) {
            v.arr.push_back(value());
            const char c = peek();
            ++i_;
            if (c == ']') break;
            if (c != ',') fail("expected , or ]");
        }
        return v;
    }
    JVal object() {
        expect('{');
        JVal v;
        v.t = JVal::Obj;
        if (peek() == '}') return ++i_, v;
        while (true) {
            std::string k = string();
            expect(':');
            v.obj.emplace_back(std::move(k), value());
            const char c = peek();
            ++i_;
            if (c == '}') break;
            if (c != ',') fail("expected , or }");
        }
        return v;
    }
};

// ----------------------------------------------------------------- files --
std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoErr("cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

uint64_t u64_le(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
    return v;
}

// WSVDMAT1 (matrix.cpp:251-284)
std::vector<double> load_matrix(const std::string& path, uint64_t& rows, uint64_t& cols) {
    const std::string buf = slurp(path);
    if (buf.size() < 24 || std::memcmp(buf.data(), "WSVDMAT1", 8) != 0) throw IoErr("not a matrix file: " + path);
    const auto* p = reinterpret_cast<const unsigned char*>(buf.data());
    rows = u64_le(p + 8);
    cols = u64_le(p + 16);
    const uint64_t n = rows * cols;
    if (buf.size() != 24 + 8 * n) throw IoErr("truncated matrix file: " + path);
    std::vector<double> v(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t bits = u64_le(p + 24 + 8 * i);
        std::memcpy(&v[i], &bits, 8);
    }
    return v;
}

// WSVDI8T1 (checkpoint.cpp:126-146)
std::vector<int8_t> load_int_matrix(const std::string& path, uint64_t& rows, uint64_t& cols) {
    const std::string buf = slurp(path);
    if (buf.size() < 24 || std::memcmp(buf.data(), "WSVDI8T1", 8) != 0)
        throw IoErr("bad int tensor magic in " + path);
    const auto* p = reinterpret_cast<const unsigned char*>(buf.data());
    rows = u64_le(p + 8);
    cols = u64_le(p + 16);
    if (buf.size() < 24 + rows * cols) throw IoErr("truncated int tensor in " + path);
    std::vector<int8_t> v(rows * cols);
    std::memcpy(v.data(), buf.data() + 24, v.size());
    return v;
}

struct Manifest {
    std::string dir;
    JVal j;
    long long E = 0, H = 0, nh = 0, nl = 0;
};

Manifest open_manifest(const char* dir) {
    if (!dir) throw IoErr("null checkpoint directory");
    Manifest m;
    m.dir = dir;
    m.j = JParser(slurp(m.dir + "/manifest.json")).parse();
    const JVal* schema = m.j.find("schema");
    if (!schema || schema->t != JVal::Str || schema->str != "wsvd-checkpoint-v1")
        throw IoErr("unsupported manifest schema in " + m.dir);
    const JVal& model = m.j.at("model");
    m.E = model.at("embed_dim").integer();
    m.H = model.at("head_dim").integer();
    m.nh = model.at("n_heads").integer();
    m.nl = model.at("n_layers").integer();
    return m;
}

const char* role_name(int role) { return role == 0 ? "q" : role == 1 ? "k" : "v"; }

const JVal& find_entry(const Manifest& m, const char* array, int layer, int head, int role) {
    if (layer < 0 || layer >= m.nl || head < 0 || head >= m.nh || role < 0 || role > 2)
        throw ShapeErr("layer / head / role out of range");
    const JVal* arr = m.j.find(array);
    if (!arr || arr->t != JVal::Arr) throw IoErr(std::string("checkpoint has no '") + array + "' entries");
    for (const JVal& e : arr->arr)
        if (e.at("layer").integer() == layer && e.at("head").integer() == head &&
            e.at("role").string() == role_name(role))
            return e;
    throw IoErr("checkpoint lacks layer " + std::to_string(layer) + " head " + std::to_string(head) + " role " +
                role_name(role));
}

}  // namespace
extern "C" void wsvd_internal_set_error(const char* msg);  // capi.cu: the wsvd_last_error() slot
namespace {

int fail(const std::exception& e) {
    g_ckpt_err = e.what();
    wsvd_internal_set_error(e.what());
    if (dynamic_cast<const ShapeErr*>(&e)) return WSVD_ESHAPE;
    return WSVD_EIO;
}

}  // namespace

extern "C" {

int wsvd_ckpt_info(const char* dir, int64_t info[8]) {
    try {
        if (!info) throw IoErr("null argument");
        const Manifest m = open_manifest(dir);
        info[0] = m.E;
        info[1] = m.H;
        info[2] = m.nh;
        info[3] = m.nl;
        const JVal* wb = m.j.find("weight_bits");
        const JVal* ab = m.j.find("activation_bits");
        info[4] = wb ? wb->integer() : 0;
        info[5] = ab ? ab->integer() : 0;
        info[6] = m.j.find("factors") ? 1 : 0;
        info[7] = m.j.find("quantized") ? 1 : 0;
        return WSVD_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int wsvd_ckpt_head(const char* dir, int32_t layer, int32_t head, int32_t role, int32_t* rank, double* a, double* b) {
    try {
        const Manifest m = open_manifest(dir);
        const JVal& e = find_entry(m, "factors", layer, head, role);
        const long long r = e.at("rank").integer();
        if (rank) *rank = static_cast<int32_t>(r);
        uint64_t ra, ca, rb, cb;
        if (a) {
            const std::vector<double> v = load_matrix(m.dir + "/" + e.at("a").string(), ra, ca);
            if (static_cast<long long>(ra) != m.E || static_cast<long long>(ca) != r)
                throw IoErr("factor shapes disagree with manifest rank");
            std::memcpy(a, v.data(), v.size() * 8);
        }
        if (b) {
            const std::vector<double> v = load_matrix(m.dir + "/" + e.at("b").string(), rb, cb);
            if (static_cast<long long>(rb) != r || static_cast<long long>(cb) != m.H)
                throw IoErr("factor shapes disagree with manifest rank");
            std::memcpy(b, v.data(), v.size() * 8);
        }
        return WSVD_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int wsvd_ckpt_head_quantized(const char* dir, int32_t layer, int32_t head, int32_t role, int32_t* rank,
                             int8_t* a_q, double* a_scales, int8_t* b_q, double* b_scales) {
    try {
        const Manifest m = open_manifest(dir);
        const JVal& e = find_entry(m, "quantized", layer, head, role);
        const long long r = e.at("rank").integer();
        if (rank) *rank = static_cast<int32_t>(r);
        auto part = [&](const JVal& w, long long rows, long long cols, int8_t* q, double* s) {
            uint64_t qr, qc, sr, sc;
            if (q) {
                const std::vector<int8_t> v = load_int_matrix(m.dir + "/" + w.at("values").string(), qr, qc);
                if (static_cast<long long>(qr) != rows || static_cast<long long>(qc) != cols)
                    throw IoErr("quantised factor shape disagrees with the manifest");
                std::memcpy(q, v.data(), v.size());
            }
            if (s) {
                const std::vector<double> v = load_matrix(m.dir + "/" + w.at("scales").string(), sr, sc);
                if (sr != 1 || static_cast<long long>(sc) != cols)
                    throw IoErr("scale row does not match integer tensor width");
                std::memcpy(s, v.data(), v.size() * 8);
            }
        };
        part(e.at("a"), m.E, r, a_q, a_scales);
        part(e.at("b"), r, m.H, b_q, b_scales);
        return WSVD_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int wsvd_ckpt_weight(const char* dir, const char* name, int64_t* rows, int64_t* cols, double* out) {
    try {
        if (!name || !rows || !cols) throw IoErr("null argument");
        const Manifest m = open_manifest(dir);
        const JVal& w = m.j.at("weights");
        const JVal* f = w.find(name);
        if (!f) throw IoErr(std::string("manifest is missing weight ") + name);
        uint64_t r, c;
        const std::vector<double> v = load_matrix(m.dir + "/" + f->string(), r, c);
        if (out) {
            if (*rows * *cols < static_cast<int64_t>(v.size())) throw ShapeErr("output buffer too small");
            std::memcpy(out, v.data(), v.size() * 8);
        }
        *rows = static_cast<int64_t>(r);
        *cols = static_cast<int64_t>(c);
        return WSVD_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// A device layer straight from a checkpoint: heads [head_begin, head_end) of
// `layer` (a head shard), quantised factors for WSVD_I8 / WSVD_I4 (the
// manifest's weight_bits must agree), fp64 factors otherwise; with
// oproj_dtype >= 0 the rows of layer<L>.w_o that multiply those heads.
int wsvd_layer_load_checkpoint(const char* dir, int32_t layer, int32_t head_begin, int32_t head_end,
                               int32_t weight_dtype, int32_t oproj_dtype, int32_t device, wsvd_layer_t* out) {
    wsvd_layer_t L = nullptr;
    try {
        if (!out) throw IoErr("null argument");
        const Manifest m = open_manifest(dir);
        if (layer < 0 || layer >= m.nl) throw ShapeErr("layer out of range");
        if (head_begin < 0 || head_end > m.nh || head_begin >= head_end) throw ShapeErr("bad head range");
        const bool quant = weight_dtype == WSVD_I8 || weight_dtype == WSVD_I4;
        if (quant) {
            const JVal* wb = m.j.find("weight_bits");
            const long long bits = wb ? wb->integer() : 0;
            if (!m.j.find("quantized")) throw IoErr("checkpoint holds no quantised factors");
            const long long want = weight_dtype == WSVD_I8 ? 8 : 4;
            if (bits != want)
                throw IoErr("requested " + std::to_string(want) + "-bit weights, the checkpoint holds " +
                            std::to_string(bits) + "-bit ones");
            // the device quantises activations per token to 8 bits (quant.cpp:131-150)
            const JVal* ab = m.j.find("activation_bits");
            if (ab && ab->integer() != 8)
                throw IoErr("checkpoint expects " + std::to_string(ab->integer()) +
                            "-bit activations; the device path quantises activations to 8 bits");
        }
        const int nh = head_end - head_begin;
        std::vector<int32_t> ranks(static_cast<size_t>(nh) * 3);
        for (int h = 0; h < nh; ++h)
            for (int role = 0; role < 3; ++role) {
                const int rc = quant ? wsvd_ckpt_head_quantized(dir, layer, head_begin + h, role, &ranks[h * 3 + role],
                                                                nullptr, nullptr, nullptr, nullptr)
                                     : wsvd_ckpt_head(dir, layer, head_begin + h, role, &ranks[h * 3 + role], nullptr,
                                                      nullptr);
                if (rc) return rc;
            }
        wsvd_layer_desc d{};
        d.embed_dim = static_cast<int32_t>(m.E);
        d.head_dim = static_cast<int32_t>(m.H);
        d.n_heads = nh;
        d.head_offset = head_begin;
        d.weight_dtype = weight_dtype;
        d.act_rotation = quant ? 1 : 0;  // "input_rotation": "hadamard" (checkpoint.cpp:220-222)
        d.device = device;
        int rc = wsvd_layer_create(&d, ranks.data(), &L);
        if (rc) {
            g_ckpt_err = wsvd_last_error();
            return rc;
        }
        for (int h = 0; h < nh; ++h)
            for (int role = 0; role < 3; ++role) {
                const int32_t r = ranks[h * 3 + role];
                if (quant) {
                    std::vector<int8_t> aq(static_cast<size_t>(m.E) * r), bq(static_cast<size_t>(r) * m.H);
                    std::vector<double> as(r), bs(m.H);
                    rc = wsvd_ckpt_head_quantized(dir, layer, head_begin + h, role, nullptr, aq.data(), as.data(),
                                                  bq.data(), bs.data());
                    if (rc) throw IoErr(g_ckpt_err);
                    rc = wsvd_layer_set_head_quantized(L, h, role, aq.data(), as.data(), bq.data(), bs.data());
                } else {
                    std::vector<double> a(static_cast<size_t>(m.E) * r), b(static_cast<size_t>(r) * m.H);
                    rc = wsvd_ckpt_head(dir, layer, head_begin + h, role, nullptr, a.data(), b.data());
                    if (rc) throw IoErr(g_ckpt_err);
                    rc = wsvd_layer_set_head(L, h, role, a.data(), b.data());
                }
                if (rc) throw IoErr(wsvd_last_error());
            }
        if (oproj_dtype >= 0) {
            const std::string name = "layer" + std::to_string(layer) + ".w_o";
            int64_t rows = m.E, cols = m.E;
            std::vector<double> wo(static_cast<size_t>(m.E) * m.E);
            rc = wsvd_ckpt_weight(dir, name.c_str(), &rows, &cols, wo.data());
            if (rc) throw IoErr(g_ckpt_err);
            if (rows != m.nh * m.H) throw IoErr("w_o rows disagree with n_heads * head_dim");
            // rows [head_begin*H, head_end*H) multiply this shard's heads (pipeline.cpp:323-329)
            const double* rows_begin = wo.data() + static_cast<size_t>(head_begin) * m.H * cols;
            rc = wsvd_layer_set_oproj(L, rows_begin, static_cast<int32_t>(cols), oproj_dtype);
            if (rc) throw IoErr(wsvd_last_error());
        }
        *out = L;
        return WSVD_OK;
    } catch (const std::exception& e) {
        if (L) wsvd_layer_destroy(L);
        return fail(e);
    }
}

}  // extern "C"
