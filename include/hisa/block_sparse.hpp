// Forwarding header: the declarations the reference keeps in hisa/block_sparse.hpp live in hisa/api.hpp.
#pragma once
#include "hisa/api.hpp"
