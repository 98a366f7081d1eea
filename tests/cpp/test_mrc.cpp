// MRC2014 I/O of the host API (include/ballmatch_b200_io.hpp) — CPU only.
// Reads files written by tests/test_cli.py (numpy) in every supported mode, byte
// order and axis order, and checks the reference's error types (volio.cpp:57-193).
#include <cmath>
#include <cstdio>
#include <string>

#include "ballmatch_b200_io.hpp"

namespace bm = ballmatch_b200;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string dir = argv[1];
    int fails = 0;
    auto check = [&](bool ok, const char* what) {
        if (!ok) {
            std::printf("FAIL %s\n", what);
            ++fails;
        }
    };
    // reference value: v(x,y,z) = x + 10 y + 100 z - 50 (written by the Python side)
    auto expect = [](int x, int y, int z) { return x + 10.0 * y + 100.0 * z - 50.0; };
    for (const char* name : {"m2_le.mrc", "m2_be.mrc", "m0.mrc", "m1.mrc", "m6.mrc", "m2_perm.mrc", "m2_ext.mrc"}) {
        const bm::Volume v = bm::read_mrc(dir + "/" + name);
        bool ok = v.n == 8;
        for (int z = 0; z < 8 && ok; ++z)
            for (int y = 0; y < 8 && ok; ++y)
                for (int x = 0; x < 8 && ok; ++x) {
                    double e = expect(x, y, z);
                    if (std::string(name) == "m0.mrc") e = static_cast<double>(static_cast<signed char>((x + y + z) % 100 - 50));
                    if (std::string(name) == "m6.mrc") e = x + 10.0 * y + 100.0 * z;
                    ok = v.at(x, y, z) == e;
                }
        check(ok, name);
    }
    check(std::fabs(bm::read_mrc(dir + "/m2_le.mrc").voxel_size - 2.5) < 1e-12, "voxel size from cella/mx");
    // write -> read round trip, single volume and stack
    bm::Volume a(8, 1.5), b(8, 1.5);
    for (size_t i = 0; i < a.data.size(); ++i) {
        a.data[i] = std::sin(0.1 * i);
        b.data[i] = std::cos(0.07 * i);
    }
    bm::write_mrc(a, dir + "/rt.mrc");
    const bm::Volume ra = bm::read_mrc(dir + "/rt.mrc");
    bool same = ra.n == 8 && std::fabs(ra.voxel_size - 1.5) < 1e-6;
    for (size_t i = 0; i < a.data.size() && same; ++i) same = ra.data[i] == static_cast<double>(static_cast<float>(a.data[i]));
    check(same, "volume round trip");
    bm::write_mrc_stack({a, b}, dir + "/rt_stack.mrc");
    const auto st = bm::read_mrc_stack(dir + "/rt_stack.mrc");
    same = st.size() == 2;
    for (size_t i = 0; i < a.data.size() && same; ++i)
        same = st[1].data[i] == static_cast<double>(static_cast<float>(b.data[i]));
    check(same, "stack round trip");
    // errors (volio.hpp:15-23)
    auto throws_as = [&](auto&& f, int kind) {
        try {
            f();
        } catch (const bm::mrc_short_read_error&) {
            return kind == 2;
        } catch (const bm::mrc_format_error&) {
            return kind == 1;
        } catch (const bm::io_error&) {
            return kind == 0;
        }
        return false;
    };
    check(throws_as([&] { bm::read_mrc(dir + "/missing.mrc"); }, 0), "missing file -> io_error");
    check(throws_as([&] { bm::read_mrc(dir + "/nostamp.mrc"); }, 1), "no MAP stamp -> mrc_format_error");
    check(throws_as([&] { bm::read_mrc(dir + "/mode3.mrc"); }, 1), "mode 3 -> mrc_format_error");
    check(throws_as([&] { bm::read_mrc(dir + "/short.mrc"); }, 2), "truncated payload -> mrc_short_read_error");
    check(throws_as([&] { bm::read_mrc(dir + "/rt_stack.mrc"); }, 1), "stack as a volume -> not cubic");
    std::printf("%d failure(s)\n", fails);
    return fails ? 1 : 0;
}
