// config_io.cpp — the reference's flat `key = value` configuration format,
// restated for demb200::SimConfig. Same keys, same rules (core/src/config_io.cpp:46-343):
// '#' comments, trimmed lines, duplicate / unknown / missing-required keys rejected with the line
// number, materials indexed in first-appearance order, contiguous wall indices, pair-restitution
// overrides; then SimConfig validation (sim_config.cpp:10-60).
#include <algorithm>
#include <cctype>
#include <charconv>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include "../../include/demb200/host.hpp"

namespace demb200 {

namespace {

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    if (b == std::string::npos) return "";
    const auto e = s.find_last_not_of(" \t\r");
    return s.substr(b, e - b + 1);
}

std::vector<std::string> split_dots(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == '.') { out.push_back(cur); cur.clear(); } else { cur += c; }
    }
    out.push_back(cur);
    return out;
}

bool identifier(const std::string& s) {
    if (s.empty() || !(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_')) return false;
    for (unsigned char c : s)
        if (!(std::isalnum(c) || c == '_')) return false;
    return true;
}

class KeyValueFile {
  public:
    KeyValueFile(const std::string& text, std::string origin) : origin_(std::move(origin)) {
        std::istringstream in(text);
        std::string raw;
        int no = 0;
        while (std::getline(in, raw)) {
            ++no;
            const auto hash = raw.find('#');
            std::string line = trim(hash == std::string::npos ? raw : raw.substr(0, hash));
            if (line.empty()) continue;
            const auto eq = line.find('=');
            if (eq == std::string::npos) fail(no, "expected 'key = value'");
            const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
            if (key.empty()) fail(no, "empty key");
            if (value.empty()) fail(no, "empty value for key '" + key + "'");
            if (values_.count(key)) fail(no, "duplicate key '" + key + "'");
            values_[key] = {no, value};
            keys_.push_back(key);
        }
    }

    [[noreturn]] void fail(int line, const std::string& what) const {
        throw ConfigError(origin_ + ":" + std::to_string(line) + ": " + what);
    }
    [[noreturn]] void fail_key(const std::string& what) const { throw ConfigError(origin_ + ": " + what); }

    struct Value {
        int line;
        std::string text;
    };
    const Value* get(const std::string& key) {
        const auto it = values_.find(key);
        if (it == values_.end()) return nullptr;
        consumed_.insert(key);
        return &it->second;
    }
    bool has(const std::string& key) const { return values_.count(key) != 0; }
    const std::vector<std::string>& keys() const { return keys_; }
    int line_of(const std::string& key) const { return values_.at(key).line; }
    void consume(const std::string& key) { consumed_.insert(key); }

    double number(const Value& v, const std::string& key) const {
        double out = 0.0;
        const char* b = v.text.data();
        const char* e = b + v.text.size();
        const auto r = std::from_chars(b, e, out);
        if (r.ec != std::errc{} || r.ptr != e) fail(v.line, "key '" + key + "': expected a number, got '" + v.text + "'");
        return out;
    }
    std::int64_t integer(const Value& v, const std::string& key) const {
        std::int64_t out = 0;
        const char* b = v.text.data();
        const char* e = b + v.text.size();
        const auto r = std::from_chars(b, e, out);
        if (r.ec != std::errc{} || r.ptr != e) fail(v.line, "key '" + key + "': expected an integer, got '" + v.text + "'");
        return out;
    }
    Vec3 vector3(const Value& v, const std::string& key) const {
        std::string t = v.text;
        std::replace(t.begin(), t.end(), ',', ' ');
        std::istringstream in(t);
        std::vector<std::string> parts;
        for (std::string p; in >> p;) parts.push_back(p);
        const std::string msg = "key '" + key + "': expected three numbers, got '" + v.text + "'";
        if (parts.size() != 3) fail(v.line, msg);
        double c[3];
        for (int k = 0; k < 3; ++k) {
            const char* b = parts[k].data();
            const char* e = b + parts[k].size();
            const auto r = std::from_chars(b, e, c[k]);
            if (r.ec != std::errc{} || r.ptr != e) fail(v.line, msg);
        }
        return Vec3{c[0], c[1], c[2]};
    }

    void read(const std::string& key, double& dst) { if (auto* v = get(key)) dst = number(*v, key); }
    template <typename T>
    void read_int(const std::string& key, T& dst) { if (auto* v = get(key)) dst = static_cast<T>(integer(*v, key)); }

    std::vector<std::string> unconsumed() const {
        std::vector<std::string> out;
        for (const auto& k : keys_)
            if (!consumed_.count(k)) out.push_back(k);
        return out;
    }
    const std::string& origin() const { return origin_; }

  private:
    std::string origin_;
    std::map<std::string, Value> values_;
    std::vector<std::string> keys_;
    std::set<std::string> consumed_;
};

void read_materials(KeyValueFile& f, SimConfig& cfg) {
    std::vector<std::string> names;  // first appearance fixes the index
    for (const auto& key : f.keys()) {
        const auto parts = split_dots(key);
        if (parts.size() == 3 && parts[0] == "material") {
            if (!identifier(parts[1])) f.fail(f.line_of(key), "bad material name '" + parts[1] + "'");
            if (std::find(names.begin(), names.end(), parts[1]) == names.end()) names.push_back(parts[1]);
        }
    }
    for (const auto& n : names) {
        MaterialParams m;
        const std::string p = "material." + n + ".";
        f.read(p + "poisson", m.poisson_ratio);
        f.read(p + "shear_modulus", m.shear_modulus);
        f.read(p + "youngs_modulus", m.youngs_modulus);
        f.read(p + "restitution", m.restitution);
        f.read(p + "mu_d", m.sliding_friction);
        cfg.materials.add(n, m);
    }
}

void read_scalars(KeyValueFile& f, SimConfig& cfg) {
    f.read("dt", cfg.dt);
    f.read("gravity.x", cfg.gravity.x);
    f.read("gravity.y", cfg.gravity.y);
    f.read("gravity.z", cfg.gravity.z);
    f.read("domain.min.x", cfg.domain_min.x);
    f.read("domain.min.y", cfg.domain_min.y);
    f.read("domain.min.z", cfg.domain_min.z);
    f.read("domain.max.x", cfg.domain_max.x);
    f.read("domain.max.y", cfg.domain_max.y);
    f.read("domain.max.z", cfg.domain_max.z);
    f.read("grid.cell_size", cfg.grid_cell_size);
    f.read_int("contacts.capacity", cfg.contact_capacity);
    f.read_int("seed", cfg.seed);
    f.read_int("simt.warp_size", cfg.warp.warp_size);
    f.read("simt.c_check", cfg.warp.c_check);
    f.read("simt.c_force", cfg.warp.c_force);
    f.read("simt.c_store", cfg.warp.c_store);
    f.read("simt.c_load", cfg.warp.c_load);
    f.read_int("run.steps", cfg.run.steps);
    f.read_int("run.warmup_steps", cfg.run.warmup_steps);
    f.read_int("run.snapshot_every", cfg.run.snapshot_every);
    if (auto* v = f.get("run.collide_variant")) {
        if (v->text == "baseline") cfg.run.collide_variant = CollideVariant::baseline;
        else if (v->text == "two_phase") cfg.run.collide_variant = CollideVariant::two_phase;
        else f.fail(v->line, "run.collide_variant must be 'baseline' or 'two_phase'");
    }
    f.read_int("particles.count", cfg.particles.count);
    f.read("particles.radius", cfg.particles.radius);
    f.read("particles.mass", cfg.particles.mass);
    if (auto* v = f.get("particles.material")) cfg.particles.material = v->text;
    if (auto* v = f.get("particles.init")) {
        if (v->text == "lattice") cfg.particles.mode = InitMode::lattice;
        else if (v->text == "headon") cfg.particles.mode = InitMode::headon;
        else f.fail(v->line, "particles.init must be 'lattice' or 'headon'");
    }
    f.read("particles.jitter", cfg.particles.jitter);
    f.read("particles.lattice_spacing", cfg.particles.lattice_spacing);
    f.read("particles.headon_gap", cfg.particles.headon_gap);
    f.read("particles.headon_speed", cfg.particles.headon_speed);
}

void read_walls(KeyValueFile& f, SimConfig& cfg) {
    std::set<int> rect, line;
    for (const auto& key : f.keys()) {
        const auto parts = split_dots(key);
        if (parts.size() != 4 || parts[0] != "wall") continue;
        int idx = -1;
        const auto r = std::from_chars(parts[2].data(), parts[2].data() + parts[2].size(), idx);
        if (r.ec != std::errc{} || r.ptr != parts[2].data() + parts[2].size() || idx < 0)
            f.fail(f.line_of(key), "bad wall index in '" + key + "'");
        if (parts[1] == "rect") rect.insert(idx);
        else if (parts[1] == "line") line.insert(idx);
        else f.fail(f.line_of(key), "unknown wall kind '" + parts[1] + "'");
    }
    auto contiguous = [&](const std::set<int>& s, const char* kind) {
        int expect = 0;
        for (int i : s)
            if (i != expect++)
                f.fail_key(std::string("wall.") + kind + " indices must be 0.." + std::to_string(static_cast<int>(s.size()) - 1));
    };
    contiguous(rect, "rect");
    contiguous(line, "line");
    auto vec = [&](const std::string& key) {
        auto* v = f.get(key);
        if (!v) f.fail_key("missing required key '" + key + "'");
        return f.vector3(*v, key);
    };
    auto mat = [&](const std::string& key) -> std::uint32_t {
        auto* v = f.get(key);
        if (!v) f.fail_key("missing required key '" + key + "'");
        if (!cfg.materials.contains(v->text)) f.fail(v->line, "key '" + key + "': unknown material '" + v->text + "'");
        return cfg.materials.index_of(v->text);
    };
    for (int i = 0; i < static_cast<int>(rect.size()); ++i) {
        const std::string p = "wall.rect." + std::to_string(i) + ".";
        RectWall w;
        w.corner = vec(p + "corner");
        w.edge_u = vec(p + "edge_u");
        w.edge_v = vec(p + "edge_v");
        w.material_id = mat(p + "material");
        cfg.rect_walls.push_back(w);
    }
    for (int i = 0; i < static_cast<int>(line.size()); ++i) {
        const std::string p = "wall.line." + std::to_string(i) + ".";
        LineWall w;
        w.a = vec(p + "a");
        w.b = vec(p + "b");
        w.material_id = mat(p + "material");
        cfg.line_walls.push_back(w);
    }
}

void read_pair_overrides(KeyValueFile& f, SimConfig& cfg) {
    for (const auto& key : f.keys()) {
        const auto parts = split_dots(key);
        if (parts.size() != 3 || parts[0] != "restitution_pair") continue;
        auto* v = f.get(key);
        if (!cfg.materials.contains(parts[1]) || !cfg.materials.contains(parts[2]))
            f.fail(v->line, "restitution_pair references an unknown material");
        cfg.materials.set_pair_restitution(cfg.materials.index_of(parts[1]), cfg.materials.index_of(parts[2]),
                                           f.number(*v, key));
    }
}

double vnorm(const Vec3& a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

}  // namespace

void validate_config(const SimConfig& cfg) {  // sim_config.cpp:10-60
    if (!(cfg.dt > 0.0)) throw ConfigError("dt: must be > 0");
    if (!(std::isfinite(cfg.gravity.x) && std::isfinite(cfg.gravity.y) && std::isfinite(cfg.gravity.z)))
        throw ConfigError("gravity: must be finite");
    const Vec3 ext{cfg.domain_max.x - cfg.domain_min.x, cfg.domain_max.y - cfg.domain_min.y, cfg.domain_max.z - cfg.domain_min.z};
    if (!(ext.x > 0.0 && ext.y > 0.0 && ext.z > 0.0)) throw ConfigError("domain: min must be strictly below max on every axis");
    if (cfg.materials.size() == 0) throw ConfigError("no materials defined");
    for (std::uint32_t k = 0; k < cfg.materials.size(); ++k) {
        const auto& m = cfg.materials.params(k);
        const std::string w = "material." + cfg.materials.name(k) + ".";
        if (!(m.poisson_ratio >= 0.0 && m.poisson_ratio < 0.5)) throw ConfigError(w + "poisson: must satisfy 0 <= sigma < 0.5");
        if (!(m.shear_modulus > 0.0)) throw ConfigError(w + "shear_modulus: must be > 0");
        if (!(m.youngs_modulus > 0.0)) throw ConfigError(w + "youngs_modulus: must be > 0");
        if (!(m.restitution > 0.0 && m.restitution <= 1.0)) throw ConfigError(w + "restitution: must satisfy 0 < eps <= 1");
        if (!(m.sliding_friction >= 0.0)) throw ConfigError(w + "mu_d: must be >= 0");
    }
    if (cfg.particles.count == 0) throw ConfigError("particles.count: must be >= 1");
    if (!(cfg.particles.radius > 0.0)) throw ConfigError("particles.radius: must be > 0");
    if (!(cfg.particles.mass > 0.0)) throw ConfigError("particles.mass: must be > 0");
    if (!cfg.materials.contains(cfg.particles.material))
        throw ConfigError("particles.material: unknown material '" + cfg.particles.material + "'");
    if (cfg.particles.mode == InitMode::headon && cfg.particles.count != 2)
        throw ConfigError("particles.count: init=headon requires exactly 2 particles");
    if (cfg.particles.lattice_spacing != 0.0 && !(cfg.particles.lattice_spacing > 2.0 * cfg.particles.radius))
        throw ConfigError("particles.lattice_spacing: must exceed the particle diameter");
    if (cfg.grid_cell_size < 0.0) throw ConfigError("grid.cell_size: must be > 0");
    if (cfg.contact_capacity < 1) throw ConfigError("contacts.capacity: must be >= 1");
    if (cfg.warp.warp_size < 1) throw ConfigError("simt.warp_size: must be >= 1");
    if (cfg.run.steps < 0) throw ConfigError("run.steps: must be >= 0");
    if (cfg.run.warmup_steps < 0) throw ConfigError("run.warmup_steps: must be >= 0");
    if (cfg.run.snapshot_every < 0) throw ConfigError("run.snapshot_every: must be >= 0");
    for (std::size_t i = 0; i < cfg.rect_walls.size(); ++i) {
        const auto& w = cfg.rect_walls[i];
        const std::string where = "wall.rect." + std::to_string(i);
        const double lu = vnorm(w.edge_u), lv = vnorm(w.edge_v);
        if (!(lu > 0.0) || !(lv > 0.0)) throw ConfigError(where + ": degenerate rectangle (zero-length edge)");
        const double d = w.edge_u.x * w.edge_v.x + w.edge_u.y * w.edge_v.y + w.edge_u.z * w.edge_v.z;
        if (std::abs(d) > 1e-9 * lu * lv) throw ConfigError(where + ": edge_u and edge_v must be orthogonal");
        if (w.material_id >= cfg.materials.size()) throw ConfigError(where + ": bad material");
    }
    for (std::size_t i = 0; i < cfg.line_walls.size(); ++i) {
        const auto& w = cfg.line_walls[i];
        const std::string where = "wall.line." + std::to_string(i);
        if (!(vnorm(Vec3{w.b.x - w.a.x, w.b.y - w.a.y, w.b.z - w.a.z}) > 0.0)) throw ConfigError(where + ": zero-length segment");
        if (w.material_id >= cfg.materials.size()) throw ConfigError(where + ": bad material");
    }
}

std::uint32_t particle_material_id(const SimConfig& cfg) { return cfg.materials.index_of(cfg.particles.material); }

SimConfig parse_config_text(const std::string& text, const std::string& origin) {
    KeyValueFile f(text, origin);
    SimConfig cfg;
    read_materials(f, cfg);
    read_scalars(f, cfg);
    read_walls(f, cfg);
    read_pair_overrides(f, cfg);
    for (const auto& key : f.unconsumed()) f.fail(f.line_of(key), "unknown key '" + key + "'");
    for (const char* req : {"dt", "particles.count", "particles.radius", "particles.mass", "particles.material"})
        if (!f.has(req)) f.fail_key(std::string("missing required key '") + req + "'");
    for (const char* axis : {"x", "y", "z"})
        for (const char* side : {"min", "max"}) {
            const std::string key = std::string("domain.") + side + "." + axis;
            if (!f.has(key)) f.fail_key("missing required key '" + key + "'");
        }
    if (cfg.materials.size() == 0) f.fail_key("no material.<name>.* block defined");
    validate_config(cfg);
    return cfg;
}

SimConfig parse_config(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError("cannot open config file " + path.string());
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_config_text(ss.str(), path.string());
}

}  // namespace demb200
