// Drop-in check of include/sfctr_b200.hpp: the reference's own C++ types go in,
// and the device path must agree with the reference's own functions
// (sfctr::SyntheticGenerator::generate, sfctr::virtual_sparse_id from the
// reference TUs in oracle/_ref/libsfctr_ref.so). Exit 0 = identical.
#include <cstdio>
#include <fstream>
#include <random>

#include "sfctr/cache_buffer.hpp"
#include "sfctr/criteo.hpp"
#include "sfctr/generator.hpp"
#include "sfctr/vsi.hpp"
#include "sfctr_b200.hpp"

int main() {
  sfctr::SimConfig rc;  // the reference's config type
  rc.num_workers = 2;
  rc.batch_size_per_worker = 512;
  rc.num_fields = 26;
  rc.vocabulary_size = 1000000;
  rc.zipf_exponent = 1.2;
  sfctr::b200::Config bc;
  bc.set("workers", "2").set("batch_size", "512").set("fields", "26").set("vocab", "1000000");
  bc.set("zipf", "1.2");
  sfctr::SyntheticGenerator ref_gen(rc);
  sfctr::b200::Generator dev_gen(bc);
  for (int step = 0; step < 3; ++step) {
    const sfctr::RawBatch a = ref_gen.generate(step);
    const sfctr::RawBatch b = dev_gen.generate(step);
    if (a.features != b.features || a.labels != b.labels) {
      std::printf("generator mismatch at step %d\n", step);
      return 1;
    }
    const sfctr::DedupBatch da = sfctr::virtual_sparse_id(a, 2);
    const sfctr::DedupBatch db = sfctr::b200::virtual_sparse_id(b, 2, 0, rc.vocabulary_size);
    if (da.global_ids != db.global_ids || da.virtual_ids != db.virtual_ids ||
        da.labels != db.labels || da.worker_row_ranges.size() != db.worker_row_ranges.size()) {
      std::printf("vsi mismatch at step %d\n", step);
      return 1;
    }
  }
  // CacheBuffer + HostStore: the reference's own classes vs the device ones, same ops
  {
    sfctr::CacheBuffer rcb(8, 4);
    sfctr::HostStore rhs(7, 4);
    sfctr::b200::CacheBuffer dcb(8, 4, 7, 1000);
    std::mt19937_64 rng(11);
    for (int i = 0; i < 600; ++i) {
      const sfctr::FeatureId f{rng() % 20};
      const std::int64_t step = i / 3;
      const int op = static_cast<int>(rng() % 5);
      int ra = 0, da = 0;  // 0 ok, 1 threw LogicError
      std::uint64_t rs = 0, ds = 0;
      if (op <= 1) {
        try { rs = rcb.admit(f, rhs.take(f), step).value; } catch (const sfctr::LogicError&) { ra = 1; }
        try { ds = dcb.admit(f, step).value; } catch (const sfctr::LogicError&) { da = 1; }
      } else if (op == 2) {
        try {
          rcb.set_needed_soon(f, false);
          rhs.put(f, rcb.evict(f));
        } catch (const sfctr::LogicError&) { ra = 1; }
        try {
          dcb.set_needed_soon(f, false);
          const sfctr::ParamEntry e = dcb.evict(f);
          const sfctr::ParamEntry& r = rhs.peek(f);
          for (std::size_t k = 0; k < r.data.size(); ++k)
            if (static_cast<float>(r.data[k]) != static_cast<float>(e.data[k])) {
              std::printf("evicted row mismatch\n");
              return 1;
            }
        } catch (const sfctr::LogicError&) { da = 1; }
      } else if (op == 3) {
        try { rcb.touch(f, step); } catch (const sfctr::LogicError&) { ra = 1; }
        try { dcb.touch(f, step); } catch (const sfctr::LogicError&) { da = 1; }
      } else {
        try { rcb.pin(f); rcb.unpin(f); } catch (const sfctr::LogicError&) { ra = 1; }
        try { dcb.pin(f); dcb.unpin(f); } catch (const sfctr::LogicError&) { da = 1; }
      }
      if (ra != da || rs != ds || rcb.free_count() != dcb.free_count() ||
          rcb.resident(f) != dcb.resident(f)) {
        std::printf("cache mismatch at op %d (op %d f %llu): %d/%d %llu/%llu\n", i, op,
                    static_cast<unsigned long long>(f.value), ra, da,
                    static_cast<unsigned long long>(rs), static_cast<unsigned long long>(ds));
        return 1;
      }
    }
    if (rcb.occupancy_diagnostics() != dcb.occupancy_diagnostics()) {
      std::printf("occupancy mismatch: %s vs %s\n", rcb.occupancy_diagnostics().c_str(),
                  dcb.occupancy_diagnostics().c_str());
      return 1;
    }
  }
  // the reference exception classes come through the façade
  try {
    sfctr::RawBatch bad;
    bad.rows = 3;
    bad.fields = 1;
    bad.features = {sfctr::FeatureId{1}, sfctr::FeatureId{2}, sfctr::FeatureId{3}};
    bad.labels = {0, 0, 0};
    sfctr::b200::virtual_sparse_id(bad, 2);
    std::printf("expected LogicError\n");
    return 1;
  } catch (const sfctr::LogicError&) {
  }
  try {
    sfctr::b200::Config c;
    c.set("workers", "0").validate();
    return 1;
  } catch (const sfctr::ConfigError&) {
  }
  // CriteoReader: the reference's own reader vs the device reader on one generated file
  {
    const char* path = "/tmp/sfctr_facade_criteo.tsv";
    std::mt19937_64 rng(3);
    std::ofstream out(path, std::ios::binary);
    for (int r = 0; r < 500; ++r) {
      out << (rng() & 1);
      for (int c = 0; c < 13; ++c) out << '\t' << (rng() % 3 ? std::to_string(rng() % 999) : "");
      for (int c = 0; c < 26; ++c) {
        out << '\t';
        if (rng() % 10) out << std::hex << (rng() & 0xffffffffu) << std::dec;
      }
      out << (r % 7 == 0 ? "\r\n" : "\n");
      if (r % 50 == 0) out << "\n";
    }
    out.close();
    sfctr::SimConfig cc = rc;
    cc.num_fields = 26;
    cc.batch_size_per_worker = 96;
    sfctr::b200::Config cb = bc;
    cb.set("batch_size", "96");
    sfctr::CriteoReader ref_rd(path, cc);
    sfctr::b200::CriteoReader dev_rd(path, cb);
    if (ref_rd.row_count() != dev_rd.row_count()) {
      std::printf("criteo row count mismatch\n");
      return 1;
    }
    for (int step = 0; step < 4; ++step) {
      const sfctr::RawBatch a = ref_rd.read_batch(step), b = dev_rd.read_batch(step);
      if (a.features != b.features || a.labels != b.labels) {
        std::printf("criteo batch mismatch at step %d\n", step);
        return 1;
      }
    }
    if (sfctr::CriteoReader::token_hash("68fd1e64") !=
        sfctr::b200::CriteoReader::token_hash("68fd1e64"))
      return 1;
  }
  sfctr::b200::Trainer tr(bc);
  const double loss = tr.step(0, dev_gen.generate(0));
  std::printf("facade ok: loss %.6f\n", loss);
  return 0;
}
