# chunking x search-on-records sweep (C5, 1M roots)
S='[{}, {"TGL_SEARCH_RECS":1}, {"TGL_CHUNK_TILES":2048}, {"TGL_CHUNK_TILES":2048,"TGL_SEARCH_RECS":1}, {"TGL_CHUNK_TILES":1024,"TGL_SEARCH_RECS":1}, {"TGL_CHUNK_TILES":512,"TGL_SEARCH_RECS":1}]'
python tools/sweep.py --settings "$S" 2>&1 | grep handle
python tools/sweep.py --roots 4194304 --reps 5 --settings "$S" 2>&1 | grep handle
