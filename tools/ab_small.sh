# same-box A/B of small-solve library builds: default and every abx/*.so, twice, interleaved
for rep in 1 2; do
for v in "" abx/*.so; do
  echo "== ${v:-default}"
  OTK_LIB=$v python tools/cfg1_profile.py 2>&1 | tail -4
done
done
nvidia-smi --query-gpu=uuid,pci.bus_id,clocks.sm,clocks.mem,clocks.gr,clocks.video,pstate,power.draw,clocks_throttle_reasons.active --format=csv
nvidia-smi -q -d CLOCK | sed -n 1,40p
