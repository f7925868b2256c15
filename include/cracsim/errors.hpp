// Forwarding header: the reference's errors.hpp surface lives in base.hpp here.
#pragma once
#include "cracsim/base.hpp"
