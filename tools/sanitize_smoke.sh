# compute-sanitizer memcheck and racecheck over the smoke configuration (the
# mbarrier / TMEM pipelines of every kernel at a small size); logs under gpurun_out/
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
