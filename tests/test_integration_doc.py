"""The ctypes stub in INTEGRATION.md mirrors the C ABI struct layout (a stale stub would make the
library read garbage past the caller's struct)."""
import os
import re

from paper_1703_08015_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_stub_desc_fields_match_binding():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = doc[doc.index("class Desc(C.Structure):"):doc.index("types = np.ones")]
    names = re.findall(r'\("([a-z_0-9]+)",', block)
    assert names == [f[0] for f in _native.DevDesc._fields_]


def test_header_desc_fields_match_binding():
    hdr = open(os.path.join(ROOT, "include", "splbm_b200.h")).read()
    body = hdr[hdr.index("typedef struct {\n  /* Geometry"):hdr.index("} splbm_dev_desc;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        for part in decl.split(","):
            m = re.search(r"\**([a-z_0-9]+)(\[\d+\])?\s*$", part.strip())
            names.append(m.group(1))
    assert names == [f[0] for f in _native.DevDesc._fields_]
