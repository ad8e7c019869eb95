# tensor-core kernel: efficiency vs item length (fixed per-tile cost?)
cd $GRAFT_REPO_ROOT
timeout 600 python tools/attn_sweep.py --case "len" --custom "len16:32,32,8,128,8192,15,2" --custom "len32:32,32,8,128,8192,31,2" --custom "len64:32,32,8,128,8192,63,2" --custom "len100:32,32,8,128,4096,99,2" --custom "len127:32,32,8,128,4096,126,2" --custom "len250:32,32,8,128,2048,249,2" --custom "len500:32,32,8,128,1024,499,2" 2>&1 | grep case
S3_TC_PACK=0 timeout 600 python tools/attn_sweep.py --case "len" --custom "len16 nopack:32,32,8,128,8192,15,2" --custom "len32 nopack:32,32,8,128,8192,31,2" --custom "len64 nopack:32,32,8,128,8192,63,2" 2>&1 | grep case
