# memcheck API report on the first os_encode launch: does an earlier runtime call avoid it?
cd $GRAFT_REPO_ROOT
cat > /tmp/f.py <<'PY'
import ctypes, sys, torch
x = torch.arange(1000, dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
L = ctypes.CDLL(sys.argv[1])
L.os_stream_check.argtypes = [ctypes.c_void_p]
print("check", L.os_stream_check(torch.cuda.current_stream().cuda_stream))
L.os_encode.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
print("rc", L.os_encode(x.data_ptr(), y.data_ptr(), 1000, 3, None))
PY
LIB=$PWD/paper_2206_01784_b200/_lib/libonesweep_b200.so
echo "== f: $(compute-sanitizer --tool memcheck python /tmp/f.py $LIB 2>&1 | grep -E 'ERROR SUMMARY|Host Frame: osb|INVALID' | head -3)"
