run() { for b in 1024 2048; do timeout 300 python bench.py --no-cpu --batch $b --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('b$b', round(d['value']), round(d['ms_per_step']*1e3,1), [(p['layer'], round(p['us'],1)) for p in r['per_layer']])"; done; }
echo "== chunked"; run
sed -i "s/constexpr std::size_t kPrefillBTileL2 = std::size_t(64) << 20;/constexpr std::size_t kPrefillBTileL2 = std::size_t(4096) << 20;/" paper_2402_04396_b200/csrc/capi.cpp
make -s -j16 -C paper_2402_04396_b200/csrc >/dev/null 2>&1 || echo BUILD FAILED
echo "== unchunked"; run
